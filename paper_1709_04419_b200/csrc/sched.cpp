// Ready-queue schedule of a planned phase (see sched.h).
#include "sched.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "api_util.h"

namespace hm {

int rq_queue_of(int lvl, bool coop) {
    // scan order: [coop 0, single 0..3, coop 1, single 4..7, coop 2, ...]
    const int per = RQ_NSINGLE / RQ_NCOOP;
    const int band = lvl / per;
    return coop ? band * (per + 1) : band * (per + 1) + 1 + (lvl % per);
}

namespace {

// rough task durations (microseconds on one CTA) for the bottom-level priority;
// only their ratios matter (trace-calibrated, tools/trace_analyze.py)
double vm_cost(const Phase& p, const VTask& v) {
    // measured at n = 64k (tools/trace_analyze.py): a one-term VM_MGEMM_ST task ~10 us,
    // ~3 us per further term; tile loads ~1.5 us; POTRF + TRTRI ~20 us
    double c = 6.0;
    for (int k = 0; k < v.ins_count; ++k) {
        const VIns& I = p.ins[v.ins_begin + k];
        switch (I.op) {
            case VM_MGEMM: c += 1.0 + 3.0 * I.ld; break;
            case VM_MGEMM_ST: c += 1.0 + 3.0 * I.t1; break;
            case VM_POTRF: case VM_TRTRI: c += 10.0; break;
            case VM_GEMM: case VM_TRSM_RLT: case VM_TRSM_LN: case VM_TRMM_LN: c += 4.0; break;
            case VM_LD: c += 1.5; break;
            default: c += 0.5; break;
        }
    }
    return c;
}

double tr_cost(const TTask& t, int nsub) {
    return 100.0 + 0.01 * (double)(t.m + t.q) * (double)t.kmax_tot / std::max(nsub, 1);
}

}  // namespace

void build_sched(const Phase& p, Sched& s) {
    const int nx = (int)p.xt.size();
    s.succ_begin.assign(nx + 1, 0);
    s.need.assign(nx, 0);
    s.queue.assign(nx, -1);
    s.slot_init.assign(nx, -1);
    s.succ2.clear();
    s.qbase.assign(RQ_NQ + 1, 0);
    s.ctl_init.assign(2 * RQ_NQ + 2, 0);
    s.succ.clear();
    if (nx == 0) return;
    // node (group leader or single task) of every task
    std::vector<int32_t> node(nx);
    for (int i = 0; i < nx; ++i) {
        const XTask& x = p.xt[i];
        node[i] = i - x.sub;
        if (x.sub < 0 || x.sub >= std::max(x.nsub, 1) || node[i] < 0 || p.xt[node[i]].nsub != x.nsub)
            throw ApiError(HM_ERR_ARG, "schedule: malformed cooperative group");
    }
    // predecessor sets of the nodes (union over a group's subs), deduplicated
    std::vector<std::pair<int32_t, int32_t>> edges;   // (pred task, successor node)
    edges.reserve(p.xdeps.size());
    for (int i = 0; i < nx; ++i) {
        const XTask& x = p.xt[i];
        for (int d = 0; d < x.dep_count; ++d) {
            const int32_t q = p.xdeps[x.dep_begin + d];
            if (q < 0 || q >= i || node[q] == node[i]) throw ApiError(HM_ERR_ARG, "schedule: dependency not topological");
            edges.push_back({q, node[i]});
        }
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    s.succ.resize(edges.size());
    for (const auto& e : edges) ++s.succ_begin[e.first + 1];
    for (int i = 0; i < nx; ++i) s.succ_begin[i + 1] += s.succ_begin[i];
    {
        std::vector<int32_t> fill(s.succ_begin.begin(), s.succ_begin.end() - 1);
        for (const auto& e : edges) {
            s.succ[fill[e.first]++] = e.second;
            ++s.need[e.second];
        }
    }
    // bottom level of every node: its cost plus the longest successor chain
    std::vector<double> bl(nx, 0.0);
    double bmax = 0.0;
    for (int i = nx - 1; i >= 0; --i) {
        const XTask& x = p.xt[i];
        double c = (x.kind == 0) ? vm_cost(p, p.vt[x.idx]) : tr_cost(p.tt[x.idx], x.nsub);
        double tail = 0.0;
        for (int k = s.succ_begin[i]; k < s.succ_begin[i + 1]; ++k) tail = std::max(tail, bl[s.succ[k]]);
        bl[i] = std::max(bl[i], c + tail);   // a leader already holds the maximum over its subs
        if (x.sub > 0) bl[node[i]] = std::max(bl[node[i]], bl[i]);   // leader (smaller index) sees its group
    }
    for (int i = 0; i < nx; ++i)
        if (node[i] == i) bmax = std::max(bmax, bl[i]);
    if (std::getenv("HM_PLAN_VERBOSE")) {
        double work = 0.0;
        for (int i = 0; i < nx; ++i) {
            const XTask& x = p.xt[i];
            work += (x.kind == 0) ? vm_cost(p, p.vt[x.idx]) : tr_cost(p.tt[x.idx], x.nsub);
        }
        std::fprintf(stderr, "sched: %d tasks, critical path %.1f ms, work %.1f CTA-ms (model)\n", nx, 1e-3 * bmax,
                     1e-3 * work);
    }
    // priority level -> queue; count slots per queue
    std::vector<int32_t> cnt(RQ_NQ, 0);
    for (int i = 0; i < nx; ++i) {
        if (node[i] != i) continue;
        const double r = bmax > 0.0 ? bl[i] / bmax : 0.0;
        int lvl = (int)std::floor((1.0 - r) * RQ_NSINGLE);
        lvl = std::min(std::max(lvl, 0), RQ_NSINGLE - 1);
        const int nsub = std::max(p.xt[i].nsub, 1);
        const int q = rq_queue_of(lvl, nsub > 1);
        s.queue[i] = q;
        cnt[q] += nsub;
    }
    for (int q = 0; q < RQ_NQ; ++q) s.qbase[q + 1] = s.qbase[q] + cnt[q];
    // roots pre-filled in their queues (a group as nsub consecutive slots)
    std::vector<int32_t> tail(RQ_NQ, 0);
    for (int i = 0; i < nx; ++i) {
        if (node[i] != i || s.need[i] != 0) continue;
        const int q = s.queue[i];
        for (int j = 0; j < std::max(p.xt[i].nsub, 1); ++j) s.slot_init[s.qbase[q] + tail[q]++] = i + j;
    }
    for (int q = 0; q < RQ_NQ; ++q) {
        s.ctl_init[2 * q] = 0;
        s.ctl_init[2 * q + 1] = tail[q];
    }
    s.max_nsub = 1;
    for (int i = 0; i < nx; ++i) s.max_nsub = std::max(s.max_nsub, p.xt[i].nsub);
    s.succ2.resize(2 * s.succ.size());
    for (size_t k = 0; k < s.succ.size(); ++k) {
        const int v = s.succ[k];
        if (s.need[v] >= (1 << (31 - RQ_NEED_SHIFT)) || p.xt[v].nsub > TR_COOP_MAX || s.queue[v] < 0)
            throw ApiError(HM_ERR_ARG, "schedule: successor does not fit the packed form");
        s.succ2[2 * k] = v;
        s.succ2[2 * k + 1] = rq_pack(s.need[v], std::max(p.xt[v].nsub, 1), s.queue[v]);
    }
    // self-check: the executor's protocol (pop, run, count arrivals, push on the
    // last one) reaches every task exactly once and fits every queue
    std::vector<int32_t> arr(nx, 0), fill(tail);
    std::vector<int32_t> work;
    for (int i = 0; i < nx; ++i)
        if (node[i] == i && s.need[i] == 0)
            for (int j = 0; j < std::max(p.xt[i].nsub, 1); ++j) work.push_back(i + j);
    size_t done = 0;
    while (done < work.size()) {
        const int i = work[done++];
        for (int k = s.succ_begin[i]; k < s.succ_begin[i + 1]; ++k) {
            const int v = s.succ[k];
            if (++arr[v] == s.need[v]) {
                const int ns = std::max(p.xt[v].nsub, 1);
                fill[s.queue[v]] += ns;
                for (int j = 0; j < ns; ++j) work.push_back(v + j);
            }
        }
    }
    bool ok = (int)work.size() == nx;
    for (int q = 0; q < RQ_NQ; ++q) ok = ok && fill[q] == s.qbase[q + 1] - s.qbase[q];
    if (!ok) throw ApiError(HM_ERR_ARG, "schedule: ready-queue replay does not reach every task");
}

}  // namespace hm

// Host planner for the H-Cholesky, forward solve and sampler (see plan.h).
//
// H-Cholesky (sec. 3.1: "L~(theta;k) is the rank-k H-matrix
// approximation of the Cholesky factor", l.263; Table 1 row "H-Cholesky",
// l.223), right-looking recursion over the cluster tree with LAZY updates:
//
//   chol(t):   chol(t0);  trsm((t1,t0), L(t0,t0));  pending(t1,t1) += (t1,t0)(t1,t0)^T;  chol(t1)
//   trsm(B=(r,s)):  X L(s,s)^T = B  recursively over the children of s;
//                   an admissible (low-rank) B = U V^T becomes U (L(s,s)^{-1} V)^T,
//                   i.e. an H forward substitution on the thin factor V.
//
// A pending update B -= X Y^T (X = (r,s), Y = (q,s)) is pushed down the
// block tree symbolically while X and Y are subdivided; when a factor is
// low-rank it becomes an explicit low-rank piece (U_x (Y V_x)^T, with Y V_x
// an H-matrix x thin product), and when the target is finally needed:
//   * a dense leaf applies all its pieces/products in one tile-VM program,
//     then POTRF (diagonal) or TRSM (off-diagonal);
//   * a low-rank block gathers [own U V^T, pieces, evaluated products] and is
//     re-truncated ONCE (QR + SVD, sigma_i > tau, tau = eps sigma^2 by default,
//     reading R4) -- the "truncated
//     low-rank updates" of the north star -- then its V is forward-solved.
// Every task declares the device regions it reads/writes (row chunks at leaf
// clusters); a task's wave is 1 + the latest wave it depends on, so each
// wave is a set of independent tasks executed by one launch per task type.
#include "plan.h"

#include <algorithm>
#include <array>
#include <climits>
#include <map>
#include <set>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <utility>

namespace hm {

int64_t Phase::n_launches() const {
    int64_t n = 0;
    for (int w = 0; w < nwaves; ++w) {
        n += (v_wave_begin[w + 1] > v_wave_begin[w]) ? 1 : 0;
        n += (t_wave_begin[w + 1] > t_wave_begin[w]) ? 1 : 0;
    }
    return n;
}

namespace {

struct LPiece {
    Thin U, V;       // U rows = cluster U.cluster, V rows = cluster V.cluster
    double alpha;
};

struct Pend {
    std::vector<std::pair<int32_t, int32_t>> prods;  // (X, Y): B -= X Y^T
    std::vector<LPiece> pieces;
};

struct Prog {
    std::vector<VIns> ins;
    std::vector<int32_t> reads, writes;
};

Dim dstat(int32_t v) { return Dim{v, -1, 0, 0}; }
Dim ddyn(int32_t stat, int32_t slot, int32_t off) { return Dim{stat, slot, off, 0}; }

struct Builder {
    const Tree& T;
    Plan& P;
    int32_t coop_max = TR_COOP_DEFAULT;   // cap of cooperative truncation groups (hm_params.coop_max)
    int64_t bump = 0;
    int32_t nres = 0;
    std::vector<int32_t> lw_wave, rd_wave;
    std::vector<int32_t> lw_task;                   // last writer task (creation id) per resource
    std::vector<std::vector<int32_t>> rd_tasks;     // readers since the last write
    std::vector<Pend> pend;
    struct XRaw { int32_t wave, kind, local; std::vector<int32_t> deps; };
    std::vector<XRaw> xraw;
    // truncation workspace ring: chunk-aligned bump allocation with wrap-around;
    // every chunk is a resource, so reuse of a region orders after its last user
    int64_t ring_chunk = 0, ring_nchunks = 0, ring_ptr = 0;
    std::vector<int32_t> ring_res;                  // resource id of each chunk (the ring can grow)
    // temporary arena for the H x thin products (Thin::tmp) and their cores: an allocation
    // lives until the last pending piece referring to it is consumed (reference count);
    // its extent then returns to a free list together with "fence" tasks (the tasks that
    // touched it), and the first access of every resource later placed on that memory
    // waits for them (pre).  Offsets are arena_base + relative offset.
    struct TmpAlloc { int64_t off, len; int32_t res0, nres, refs; };
    std::vector<TmpAlloc> tmps;
    struct Ext { int64_t len; std::vector<int32_t> fences; int32_t fwave; };
    std::map<int64_t, Ext> afree;                                  // free extents by offset
    std::vector<std::set<std::pair<int32_t, int64_t>>> aclass;     // per size class: (fence wave, off)
    int64_t arena_base = 0, arena_top = 0;
    int arena_mode = 1;   // experiments (HM_ARENA_MODE): 0 never recycle, 1 wave rule, 2 any free extent
    int64_t arena_budget = INT64_MAX;   // doubles; above it, recycling ignores the wave rule
    std::vector<std::vector<int32_t>> pre;          // per resource: tasks its first access waits for
    static constexpr size_t FENCE_MAX = 8;
    // current phase state
    Phase* ph = nullptr;
    std::vector<std::pair<int32_t, VTask>> vraw;   // (wave, task)
    std::vector<std::pair<int32_t, TTask>> traw;
    int64_t n_tasks = 0;

    Builder(const Tree& t, Plan& p) : T(t), P(p) {}

    const Cluster& C(int32_t c) const { return T.clusters[c]; }
    const Block& B(int32_t b) const { return T.blocks[b]; }

    int64_t alloc(int64_t n) {
        int64_t o = bump;
        bump += (n + 31) & ~int64_t(31);   // 256-byte alignment
        return o;
    }
    int32_t new_res(int32_t n) {
        int32_t b = nres;
        nres += n;
        lw_wave.resize(nres, -1);
        rd_wave.resize(nres, -1);
        lw_task.resize(nres, -1);
        rd_tasks.resize(nres);
        pre.resize(nres);
        return b;
    }

    void grow_ring(int64_t nchunks) {
        while ((int64_t)ring_res.size() < nchunks) ring_res.push_back(new_res(1));
        ring_nchunks = (int64_t)ring_res.size();
    }

    // ---- temporary arena ----------------------------------------------------
    // A task with no instructions that depends on `deps`: one edge per dependency
    // instead of (new users) x (old users) edges when memory is recycled.
    int32_t noop_task(std::vector<int32_t> deps) {
        std::sort(deps.begin(), deps.end());
        deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
        int32_t w = 0;
        for (int32_t d : deps) w = std::max(w, xraw[d].wave + 1);
        VTask t;
        t.ins_begin = (int32_t)ph->ins.size();
        t.ins_count = 0;
        xraw.push_back({w, 0, (int32_t)vraw.size(), std::move(deps)});
        vraw.push_back({w, t});
        ++n_tasks;
        return (int32_t)xraw.size() - 1;
    }
    void compress_fences(std::vector<int32_t>& f) {
        std::sort(f.begin(), f.end());
        f.erase(std::unique(f.begin(), f.end()), f.end());
        if (f.size() > FENCE_MAX) f = {noop_task(f)};
    }
    static int size_class(int64_t len) {   // floor(log2(len / 32))
        int c = 0;
        for (int64_t v = len >> 5; v > 1; v >>= 1) ++c;
        return c;
    }
    void ext_unlink(int64_t off, const Ext& e) { aclass[size_class(e.len)].erase({e.fwave, off}); }
    void arena_insert(int64_t off, int64_t len, std::vector<int32_t> f) {
        auto nx = afree.lower_bound(off);
        if (nx != afree.end() && nx->first == off + len) {
            len += nx->second.len;
            f.insert(f.end(), nx->second.fences.begin(), nx->second.fences.end());
            ext_unlink(nx->first, nx->second);
            afree.erase(nx);
        }
        auto pv = afree.lower_bound(off);
        if (pv != afree.begin()) {
            --pv;
            if (pv->first + pv->second.len == off) {
                off = pv->first;
                len += pv->second.len;
                f.insert(f.end(), pv->second.fences.begin(), pv->second.fences.end());
                ext_unlink(pv->first, pv->second);
                afree.erase(pv);
            }
        }
        compress_fences(f);
        int32_t fw = -1;
        for (int32_t t : f) fw = std::max(fw, xraw[t].wave);
        const int c = size_class(len);
        if ((int)aclass.size() <= c) aclass.resize(c + 1);
        aclass[c].insert({fw, off});
        afree[off] = Ext{len, std::move(f), fw};
    }
    // Allocation policy.  Recycling memory adds dependencies on the tasks that used it
    // last (its fences); those are harmless only if they finish before the new user
    // could start anyway.  The planner's proxy for "anyway" is the wave: reuse a free
    // extent only if its fences sit in an earlier wave than `wnat` (the wave of the
    // data the new allocation is computed from), oldest fences first; else grow the arena.
    int64_t arena_take(int64_t len, int32_t wnat, std::vector<int32_t>& fences) {
        len = (len + 31) & ~int64_t(31);   // 256-byte alignment
        int64_t best = -1;
        int32_t bw = INT32_MAX;
        if (arena_mode == 0) wnat = INT32_MIN;
        if (arena_mode == 2) wnat = INT32_MAX;
        // over the budget: recycle the extent with the oldest fences even if they are late
        const bool over = arena_top + len > arena_budget;
        for (int c = size_class(len); c < (int)aclass.size(); ++c) {
            int scanned = 0;
            for (const auto& e : aclass[c]) {
                if ((!over && e.first >= wnat) || e.first >= bw) break;
                if (afree[e.second].len >= len) {
                    best = e.second;
                    bw = e.first;
                    break;
                }
                if (++scanned > 16) break;
            }
        }
        if (best >= 0) {
            auto fit = afree.find(best);
            Ext e = std::move(fit->second);
            ext_unlink(best, e);
            afree.erase(fit);
            fences = e.fences;
            if (e.len > len) arena_insert(best + len, e.len - len, std::move(e.fences));
            return best;
        }
        fences.clear();
        const int64_t off = arena_top;
        arena_top += len;
        return off;
    }
    // new arena allocation of n doubles whose memory is covered by resources [res0, res0 + nres)
    double site_bytes[4] = {0, 0, 0, 0};
    int cur_site = 0;
    int32_t tmp_new(int64_t n, int32_t res0, int32_t nres, int32_t wnat, int64_t& off) {
        site_bytes[cur_site] += 8.0 * n;
        std::vector<int32_t> f;
        const int64_t rel = arena_take(n, wnat, f);
        for (int32_t r = res0; r < res0 + nres; ++r) pre[r] = f;
        tmps.push_back({rel, (n + 31) & ~int64_t(31), res0, nres, 0});
        off = arena_base + rel;
        return (int32_t)tmps.size() - 1;
    }
    void tmp_release(int32_t id) {
        const TmpAlloc a = tmps[id];
        std::vector<int32_t> f;
        for (int32_t r = a.res0; r < a.res0 + a.nres; ++r) {
            if (lw_task[r] >= 0) f.push_back(lw_task[r]);
            f.insert(f.end(), rd_tasks[r].begin(), rd_tasks[r].end());
            f.insert(f.end(), pre[r].begin(), pre[r].end());   // never accessed: keep the old fences
            pre[r].clear();
        }
        arena_insert(a.off, a.len, std::move(f));
    }
    void tmp_ref(const Thin& t, int d) {
        if (t.tmp < 0) return;
        int32_t& r = tmps[t.tmp].refs;
        r += d;
        if (r < 0) throw std::logic_error("planner: temporary released twice");
        if (r == 0) tmp_release(t.tmp);
    }
    void piece_ref(const LPiece& pc, int d) {
        tmp_ref(pc.U, d);
        tmp_ref(pc.V, d);
    }
    // phases run one after another: fences of an earlier phase are met
    void arena_new_phase() {
        std::map<int64_t, Ext> old;
        old.swap(afree);
        aclass.clear();
        for (auto& e : old) arena_insert(e.first, e.second.len, {});
        for (auto& v : pre) v.clear();
    }
    // wave after which the data in resources `rs` (a product's source) is available
    // earliest wave the product H(Yb) x V could be computed in (wave rule of arena_take)
    int32_t wnat_of(int32_t Yb, const Thin& V) const {
        return wnat_mode ? std::max(avail_block(Yb), avail_wave(V)) : avail_wave(V);
    }
    int wnat_mode = 1;
    // wave after which every block of the subtree of b (the other factor of a product) is final
    int32_t avail_block(int32_t b) const {
        const BStore& st = P.bs[b];
        if (st.kind == ST_DENSE) return lw_wave[st.d_res] + 1;
        if (st.kind == ST_LR) return std::max(avail_wave(thin_U(b)), avail_wave(thin_V(b)));
        int32_t w = 0;
        for (int i = 0; i < 4; ++i)
            if (B(b).child[i] >= 0) w = std::max(w, avail_block(B(b).child[i]));
        return w;
    }
    int32_t avail_wave(const Thin& M) const {
        int32_t w = 0;
        for (int32_t i = 0; i < P.leaf_count[M.cluster]; ++i) w = std::max(w, lw_wave[M.res0 + i] + 1);
        return w;
    }

    // ---- dependency tracking ------------------------------------------
    int32_t wave_of(const std::vector<int32_t>& reads, const std::vector<int32_t>& writes,
                    std::vector<int32_t>& deps) {
        const int32_t me = (int32_t)xraw.size();
        deps.clear();
        int32_t wpre = 0;
        // first access to memory recycled from the temporary arena: after its fences
        for (const auto* rs : {&reads, &writes})
            for (int32_t r : *rs)
                for (int32_t f : pre[r]) {
                    deps.push_back(f);
                    wpre = std::max(wpre, xraw[f].wave + 1);
                }
        for (int32_t r : writes) pre[r].clear();
        for (int32_t r : reads)
            if (lw_task[r] >= 0) deps.push_back(lw_task[r]);
        for (int32_t r : writes) {
            if (lw_task[r] >= 0) deps.push_back(lw_task[r]);
            for (int32_t x : rd_tasks[r]) deps.push_back(x);
        }
        std::sort(deps.begin(), deps.end());
        deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
        for (int32_t r : reads) rd_tasks[r].push_back(me);
        for (int32_t r : writes) {
            lw_task[r] = me;
            rd_tasks[r].clear();
        }
        int32_t w = wpre;
        for (int32_t r : reads)
            if (lw_wave[r] >= 0) w = std::max(w, lw_wave[r] + 1);
        for (int32_t r : writes) {
            if (lw_wave[r] >= 0) w = std::max(w, lw_wave[r] + 1);
            if (rd_wave[r] >= 0) w = std::max(w, rd_wave[r] + 1);
        }
        for (int32_t r : reads) rd_wave[r] = std::max(rd_wave[r], w);
        for (int32_t r : writes) {
            lw_wave[r] = w;
            rd_wave[r] = -1;
        }
        return w;
    }

    // Peephole: every "LD t1 <- A; LD t2 <- B; GEMM t0 += alpha op(t1) op(t2)" triple becomes a
    // term of one VM_MGEMM on t0 (consecutive triples on the same t0 share the instruction),
    // so the device streams the operands through a pipelined DMMA loop instead of
    // loading, synchronising and multiplying tile by tile.
    static void fuse_mgemm(const std::vector<VIns>& in, std::vector<VIns>& out, std::vector<VTerm>& terms) {
        size_t i = 0;
        while (i < in.size()) {
            auto is_triple = [&](size_t j, bool first) {
                return j + 2 < in.size() && in[j].op == VM_LD && in[j + 1].op == VM_LD && in[j + 2].op == VM_GEMM &&
                       in[j + 2].t1 == in[j].t0 && in[j + 2].t2 == in[j + 1].t0 && in[j].t0 != in[j + 1].t0 &&
                       (in[j + 2].beta == 1.0 || (first && in[j + 2].beta == 0.0)) && in[j + 2].t0 != in[j].t0 &&
                       in[j + 2].t0 != in[j + 1].t0;
            };
            if (!is_triple(i, true)) {
                out.push_back(in[i]);
                ++i;
                continue;
            }
            if (in[i + 2].beta == 0.0) {                 // C = A B: zero C (dims of op(A) x op(B)) first
                VIns z = mk(VM_ZERO);
                z.t0 = in[i + 2].t0;
                z.rows = in[i + 2].ta ? in[i].cols : in[i].rows;
                z.cols = in[i + 2].tb ? in[i + 1].rows : in[i + 1].cols;
                out.push_back(z);
            }
            VIns m = in[i + 2];
            m.op = VM_MGEMM;
            m.goff = (int64_t)terms.size();
            m.ld = 0;
            bool firstt = true;
            while (is_triple(i, firstt) && in[i + 2].t0 == m.t0 && m.ld < VM_MAX_TERMS) {
                firstt = false;
                VTerm tm{};
                tm.a_off = in[i].goff; tm.a_ld = in[i].ld; tm.a_rows = in[i].rows; tm.a_cols = in[i].cols;
                tm.b_off = in[i + 1].goff; tm.b_ld = in[i + 1].ld; tm.b_rows = in[i + 1].rows; tm.b_cols = in[i + 1].cols;
                tm.ta = in[i + 2].ta; tm.tb = in[i + 2].tb; tm.alpha = in[i + 2].alpha;
                terms.push_back(tm);
                ++m.ld;
                i += 3;
            }
            out.push_back(m);
        }
    }

    // Second peephole: "ZERO t; VM_MGEMM t; ST t -> D" and "LD t <- D; VM_MGEMM t; ST t -> D"
    // become one VM_MGEMM_ST writing the accumulators to D directly, provided no later
    // instruction reads t before redefining it.
    static bool reads_tile(const VIns& I, uint8_t t) {
        switch (I.op) {
            case VM_ST: case VM_POTRF: case VM_TRSM_RLT: case VM_TRSM_LN: case VM_TRMM_LN: case VM_MGEMM:
                return I.t0 == t || ((I.op == VM_TRSM_RLT || I.op == VM_TRSM_LN || I.op == VM_TRMM_LN) && I.t1 == t);
            case VM_GEMM: return I.t1 == t || I.t2 == t || (I.t0 == t && I.beta != 0.0);
            case VM_ADD: return I.t0 == t || I.t1 == t;
            case VM_TRTRI: return I.t1 == t;
            default: return false;
        }
    }
    static bool defines_tile(const VIns& I, uint8_t t) {
        return I.t0 == t && (I.op == VM_LD || I.op == VM_ZERO || (I.op == VM_GEMM && I.beta == 0.0));
    }
    static void fuse_mgemm_st(const std::vector<VIns>& in, std::vector<VIns>& out) {
        size_t i = 0;
        while (i < in.size()) {
            bool fused = false;
            if (i + 2 < in.size() && in[i + 1].op == VM_MGEMM && in[i + 2].op == VM_ST) {
                const VIns &a = in[i], &m = in[i + 1], &st = in[i + 2];
                const uint8_t t = m.t0;
                const bool zero_head = a.op == VM_ZERO && a.t0 == t;
                const bool ld_head = a.op == VM_LD && a.t0 == t && a.goff == st.goff && a.ld == st.ld &&
                                     std::memcmp(&a.rows, &st.rows, sizeof(Dim)) == 0 &&
                                     std::memcmp(&a.cols, &st.cols, sizeof(Dim)) == 0;
                if ((zero_head || ld_head) && st.t0 == t) {
                    bool dead = true;
                    for (size_t j = i + 3; j < in.size(); ++j) {
                        if (reads_tile(in[j], t)) { dead = false; break; }
                        if (defines_tile(in[j], t)) break;
                    }
                    if (dead) {
                        VIns f = st;
                        f.op = VM_MGEMM_ST;
                        f.t1 = (uint8_t)m.ld;            // term count (<= VM_MAX_TERMS)
                        f.pad2 = (int32_t)m.goff;        // first term
                        f.beta = ld_head ? 1.0 : 0.0;
                        out.push_back(f);
                        i += 3;
                        fused = true;
                    }
                }
            }
            if (!fused) {
                out.push_back(in[i]);
                ++i;
            }
        }
    }

    void emit_vm(Prog& pg) {
        if (pg.ins.empty()) return;
        std::sort(pg.reads.begin(), pg.reads.end());
        pg.reads.erase(std::unique(pg.reads.begin(), pg.reads.end()), pg.reads.end());
        std::sort(pg.writes.begin(), pg.writes.end());
        pg.writes.erase(std::unique(pg.writes.begin(), pg.writes.end()), pg.writes.end());
        std::vector<int32_t> deps;
        int32_t w = wave_of(pg.reads, pg.writes, deps);
        VTask t;
        t.ins_begin = (int32_t)ph->ins.size();
        {
            std::vector<VIns> tmp;
            fuse_mgemm(pg.ins, tmp, ph->terms);
            fuse_mgemm_st(tmp, ph->ins);
        }
        t.ins_count = (int32_t)ph->ins.size() - t.ins_begin;
        xraw.push_back({w, 0, (int32_t)vraw.size(), std::move(deps)});
        vraw.push_back({w, t});
        ++n_tasks;
    }

    // ---- thin matrices -------------------------------------------------
    Thin sub(const Thin& M, int32_t child) const {
        Thin s = M;
        s.off = M.off + (C(child).lo - C(M.cluster).lo);
        s.res0 = M.res0 + (P.leaf_begin[child] - P.leaf_begin[M.cluster]);
        s.cluster = child;
        return s;
    }
    int32_t chunk_res(const Thin& M, int32_t leafc) const {
        return M.res0 + (P.leaf_begin[leafc] - P.leaf_begin[M.cluster]);
    }
    void thin_res(const Thin& M, std::vector<int32_t>& out) const {
        for (int32_t i = 0; i < P.leaf_count[M.cluster]; ++i) out.push_back(M.res0 + i);
    }
    Thin new_thin(int32_t cluster, int32_t cols, int32_t slot, int32_t wnat) {
        Thin t;
        t.cluster = cluster;
        t.ld = (int32_t)C(cluster).size();
        t.cols = cols;
        t.slot = slot;
        t.res0 = new_res(P.leaf_count[cluster]);
        t.tmp = tmp_new((int64_t)t.ld * cols, t.res0, P.leaf_count[cluster], wnat, t.off);
        return t;
    }
    Thin thin_U(int32_t b) const {
        const BStore& s = P.bs[b];
        Thin t;
        t.off = s.u_off; t.ld = s.m; t.cluster = B(b).t; t.cols = s.cap; t.slot = s.rslot; t.res0 = s.u_res0;
        return t;
    }
    Thin thin_V(int32_t b) const {
        const BStore& s = P.bs[b];
        Thin t;
        t.off = s.v_off; t.ld = s.p; t.cluster = B(b).s; t.cols = s.cap; t.slot = s.rslot; t.res0 = s.v_res0;
        return t;
    }
    // dense leaf-level block viewed as a thin matrix over its row cluster
    Thin thin_D(int32_t b) const {
        const BStore& s = P.bs[b];
        Thin t;
        t.off = s.d_off; t.ld = s.m; t.cluster = B(b).t; t.cols = s.p; t.slot = -1; t.res0 = s.d_res;
        return t;
    }

    // VM instruction helpers
    static VIns mk(uint8_t op) {
        VIns i{};
        i.op = op;
        i.rows = dstat(0);
        i.cols = dstat(0);
        i.alpha = 1.0;
        i.beta = 0.0;
        return i;
    }
    // load the leaf-row chunk `leafc` of M, columns [c0, c0+64)
    void ld_thin(Prog& pg, uint8_t tile, const Thin& M, int32_t leafc, int32_t c0) {
        VIns i = mk(VM_LD);
        i.t0 = tile;
        i.rows = dstat((int32_t)C(leafc).size());
        i.cols = (M.slot >= 0) ? ddyn(std::min(64, M.cols - c0), M.slot, c0) : dstat(std::min(64, M.cols - c0));
        i.goff = M.off + (C(leafc).lo - C(M.cluster).lo) + (int64_t)c0 * M.ld;
        i.ld = M.ld;
        pg.ins.push_back(i);
        pg.reads.push_back(chunk_res(M, leafc));
    }
    void st_thin(Prog& pg, uint8_t tile, const Thin& M, int32_t leafc, int32_t c0) {
        VIns i = mk(VM_ST);
        i.t0 = tile;
        i.rows = dstat((int32_t)C(leafc).size());
        i.cols = (M.slot >= 0) ? ddyn(std::min(64, M.cols - c0), M.slot, c0) : dstat(std::min(64, M.cols - c0));
        i.goff = M.off + (C(leafc).lo - C(M.cluster).lo) + (int64_t)c0 * M.ld;
        i.ld = M.ld;
        pg.ins.push_back(i);
        pg.writes.push_back(chunk_res(M, leafc));
    }
    void ld_dense(Prog& pg, uint8_t tile, int32_t b) {
        const BStore& s = P.bs[b];
        VIns i = mk(VM_LD);
        i.t0 = tile;
        i.rows = dstat(s.m);
        i.cols = dstat(s.p);
        i.goff = s.d_off;
        i.ld = s.m;
        pg.ins.push_back(i);
        pg.reads.push_back(s.d_res);
    }
    void ld_inv(Prog& pg, uint8_t tile, int32_t d) {   // L^{-1} of diagonal leaf block d
        const BStore& s = P.bs[d];
        VIns i = mk(VM_LD);
        i.t0 = tile;
        i.rows = dstat(s.m);
        i.cols = dstat(s.m);
        i.goff = s.inv_off;
        i.ld = s.m;
        pg.ins.push_back(i);
        pg.reads.push_back(s.inv_res);
    }
    void st_dense(Prog& pg, uint8_t tile, int32_t b) {
        const BStore& s = P.bs[b];
        VIns i = mk(VM_ST);
        i.t0 = tile;
        i.rows = dstat(s.m);
        i.cols = dstat(s.p);
        i.goff = s.d_off;
        i.ld = s.m;
        pg.ins.push_back(i);
        pg.writes.push_back(s.d_res);
    }
    // small matrix (rank x width) chunk load/store; rows/cols dims given explicitly
    void ld_small(Prog& pg, uint8_t tile, int64_t off, int32_t ld, Dim rows, Dim cols, int32_t res) {
        VIns i = mk(VM_LD);
        i.t0 = tile; i.rows = rows; i.cols = cols; i.goff = off; i.ld = ld;
        pg.ins.push_back(i);
        pg.reads.push_back(res);
    }
    void st_small(Prog& pg, uint8_t tile, int64_t off, int32_t ld, Dim rows, Dim cols, int32_t res) {
        VIns i = mk(VM_ST);
        i.t0 = tile; i.rows = rows; i.cols = cols; i.goff = off; i.ld = ld;
        pg.ins.push_back(i);
        pg.writes.push_back(res);
    }
    void zero(Prog& pg, uint8_t tile, Dim rows, Dim cols) {
        VIns i = mk(VM_ZERO);
        i.t0 = tile; i.rows = rows; i.cols = cols;
        pg.ins.push_back(i);
    }
    void gemm(Prog& pg, uint8_t c, uint8_t a, bool ta, uint8_t b, bool tb, double alpha, double beta) {
        VIns i = mk(VM_GEMM);
        i.t0 = c; i.t1 = a; i.t2 = b; i.ta = ta; i.tb = tb; i.alpha = alpha; i.beta = beta;
        pg.ins.push_back(i);
    }
    void op2(Prog& pg, uint8_t op, uint8_t t0, uint8_t t1, int64_t goff = 0) {
        VIns i = mk(op);
        i.t0 = t0; i.t1 = t1; i.goff = goff;
        pg.ins.push_back(i);
    }
    Dim wdim(const Thin& M, int32_t c0) const {
        return (M.slot >= 0) ? ddyn(std::min(64, M.cols - c0), M.slot, c0) : dstat(std::min(64, M.cols - c0));
    }

    // leaf clusters under c (in order)
    void leaves_of(int32_t c, std::vector<int32_t>& out) const {
        for (int32_t i = 0; i < P.leaf_count[c]; ++i) out.push_back(P.leaf_cluster[P.leaf_begin[c] + i]);
    }

    // ---- H-matrix x thin:  Tout (+)= alpha * Y * Vsrc -------------------
    // Y: lower off-diagonal block (q, s) of any kind; Vsrc rows = s, Tout rows = q.
    void hxt(int32_t Y, const Thin& Vsrc, const Thin& Tout, double alpha, bool accumulate) {
        const int32_t W = Vsrc.cols;
        // stage A: cores of the low-rank leaves, core_b = V_b^T Vsrc|_{s_b}
        std::vector<int32_t> stack{Y}, lr_leaves;
        const int32_t noc = (W + 63) / 64;
        struct Core { int64_t off; int32_t res; int32_t tmp; };   // res: one resource per (kc, oc) chunk
        std::vector<std::pair<int32_t, Core>> cores;
        while (!stack.empty()) {
            int32_t b = stack.back();
            stack.pop_back();
            const BStore& s = P.bs[b];
            if (s.kind == ST_SUB) {
                for (int i = 0; i < 4; ++i)
                    if (B(b).child[i] >= 0) stack.push_back(B(b).child[i]);
            } else if (s.kind == ST_LR) {
                lr_leaves.push_back(b);
            }
        }
        for (int32_t b : lr_leaves) {
            const BStore& s = P.bs[b];
            Core cr;
            const int32_t nr = ((s.cap + 63) / 64) * noc;
            cr.res = new_res(nr);
            cur_site = 3;
            cr.tmp = tmp_new((int64_t)s.cap * W, cr.res, nr, std::max(avail_wave(thin_V(b)), avail_wave(Vsrc)), cr.off);
            const Thin Vb = thin_V(b);
            const Thin Vs = sub(Vsrc, B(b).s);
            std::vector<int32_t> lv;
            leaves_of(B(b).s, lv);
            for (int32_t kc = 0; kc < s.cap; kc += 64) {
                for (int32_t oc = 0; oc < W; oc += 64) {
                    Prog pg;
                    Dim rows = ddyn(std::min(64, s.cap - kc), s.rslot, kc);
                    Dim cols = wdim(Vsrc, oc);
                    zero(pg, 0, rows, cols);
                    for (int32_t c : lv) {
                        ld_thin(pg, 1, Vb, c, kc);
                        ld_thin(pg, 2, Vs, c, oc);
                        gemm(pg, 0, 1, true, 2, false, 1.0, 1.0);
                    }
                    st_small(pg, 0, cr.off + kc + (int64_t)oc * s.cap, s.cap, rows, cols,
                             cr.res + (kc / 64) * noc + oc / 64);
                    emit_vm(pg);
                }
            }
            cores.push_back({b, cr});
        }
        auto core_of = [&](int32_t b) -> Core {
            for (auto& pr : cores)
                if (pr.first == b) return pr.second;
            throw std::logic_error("core not found");
        };
        // stage B: row recursion over Y carrying the active low-rank ancestors
        struct Frame { int32_t r; std::vector<int32_t> blocks; std::vector<int32_t> active; };
        std::vector<Frame> fs;
        fs.push_back(Frame{B(Y).t, {Y}, {}});
        while (!fs.empty()) {
            Frame f = std::move(fs.back());
            fs.pop_back();
            std::vector<int32_t> sub_blocks, dense_here;
            std::vector<int32_t> active = f.active;
            for (int32_t b : f.blocks) {
                const BStore& s = P.bs[b];
                if (s.kind == ST_LR) active.push_back(b);
                else if (s.kind == ST_DENSE) dense_here.push_back(b);
                else sub_blocks.push_back(b);
            }
            const Cluster& rc = C(f.r);
            if (rc.leaf()) {
                for (int32_t oc = 0; oc < W; oc += 64) {
                    Prog pg;
                    if (accumulate) ld_thin(pg, 0, Tout, f.r, oc);
                    else zero(pg, 0, dstat((int32_t)rc.size()), wdim(Tout, oc));
                    for (int32_t b : dense_here) {
                        ld_dense(pg, 1, b);
                        ld_thin(pg, 2, sub(Vsrc, B(b).s), B(b).s, oc);
                        gemm(pg, 0, 1, false, 2, false, alpha, 1.0);
                    }
                    for (int32_t b : active) {
                        const BStore& s = P.bs[b];
                        Core cr = core_of(b);
                        const Thin Ub = thin_U(b);
                        for (int32_t kc = 0; kc < s.cap; kc += 64) {
                            ld_thin(pg, 1, Ub, f.r, kc);
                            ld_small(pg, 2, cr.off + kc + (int64_t)oc * s.cap, s.cap,
                                     ddyn(std::min(64, s.cap - kc), s.rslot, kc), wdim(Vsrc, oc),
                                     cr.res + (kc / 64) * noc + oc / 64);
                            gemm(pg, 0, 1, false, 2, false, alpha, 1.0);
                        }
                    }
                    st_thin(pg, 0, Tout, f.r, oc);
                    emit_vm(pg);
                }
                if (!sub_blocks.empty()) throw std::logic_error("hxt: subdivided block at a leaf row");
            } else {
                for (int i = 0; i < 2; ++i) {
                    Frame nf;
                    nf.r = rc.child[i];
                    nf.active = active;
                    for (int32_t b : sub_blocks) {
                        // off-diagonal block children: (r_i, s_j) = child[i + 2j]
                        for (int j = 0; j < 2; ++j) nf.blocks.push_back(B(b).child[i + 2 * j]);
                    }
                    fs.push_back(std::move(nf));
                }
            }
        }
        for (auto& pr : cores) tmp_release(pr.second.tmp);
    }

    // ---- forward substitution  V <- L(s,s)^{-1} V --------------------------
    void fsolve(int32_t s, const Thin& V) {
        const int32_t d = P.diag_of[s];
        if (C(s).leaf()) {
            // V_s <- L_ss^{-1} V_s as a product with the inverse the POTRF task stored
            for (int32_t oc = 0; oc < V.cols; oc += 64) {
                Prog pg;
                ld_inv(pg, 1, d);
                ld_thin(pg, 0, V, s, oc);
                gemm(pg, 2, 1, false, 0, false, 1.0, 0.0);
                st_thin(pg, 2, V, s, oc);
                emit_vm(pg);
            }
            return;
        }
        const int32_t s0 = C(s).child[0], s1 = C(s).child[1];
        const BStore& so = P.bs[B(d).child[1]];
        if (so.x_off >= 0) {
            // two leaves: [V0; V1] <- [L00^{-1} 0; X10 L11^{-1}] [V0; V1] in one task per column
            // chunk (V1 first: it reads the old V0)
            const Thin V0 = sub(V, s0), V1 = sub(V, s1);
            for (int32_t oc = 0; oc < V.cols; oc += 64) {
                Prog pg;
                zero(pg, 0, dstat(so.m), wdim(V, oc));
                VIns lx = mk(VM_LD);
                lx.t0 = 1; lx.rows = dstat(so.m); lx.cols = dstat(so.p); lx.goff = so.x_off; lx.ld = so.m;
                pg.ins.push_back(lx);
                pg.reads.push_back(so.x_res);
                ld_thin(pg, 2, V0, s0, oc);
                gemm(pg, 0, 1, false, 2, false, 1.0, 1.0);
                ld_inv(pg, 1, P.diag_of[s1]);
                ld_thin(pg, 2, V1, s1, oc);
                gemm(pg, 0, 1, false, 2, false, 1.0, 1.0);
                st_thin(pg, 0, V1, s1, oc);
                zero(pg, 0, dstat((int32_t)C(s0).size()), wdim(V, oc));
                ld_inv(pg, 1, P.diag_of[s0]);
                ld_thin(pg, 2, V0, s0, oc);
                gemm(pg, 0, 1, false, 2, false, 1.0, 1.0);
                st_thin(pg, 0, V0, s0, oc);
                emit_vm(pg);
            }
            return;
        }
        fsolve(s0, sub(V, s0));
        hxt(B(d).child[1], sub(V, s0), sub(V, s1), -1.0, true);
        fsolve(s1, sub(V, s1));
    }

    // ---- X <- L(t,t) X (sampler) -----------------------------------------
    void lmul(int32_t t, const Thin& X) {
        const int32_t d = P.diag_of[t];
        if (C(t).leaf()) {
            for (int32_t oc = 0; oc < X.cols; oc += 64) {
                Prog pg;
                ld_thin(pg, 0, X, t, oc);
                ld_dense(pg, 1, d);
                op2(pg, VM_TRMM_LN, 0, 1);
                st_thin(pg, 0, X, t, oc);
                emit_vm(pg);
            }
            return;
        }
        const int32_t t0 = C(t).child[0], t1 = C(t).child[1];
        lmul(t1, sub(X, t1));
        hxt(B(d).child[1], sub(X, t0), sub(X, t1), 1.0, true);
        lmul(t0, sub(X, t0));
    }

    // ---- pending updates ---------------------------------------------------
    // children of block b as (child id, i, k) with i/k the child index of its row/col cluster
    void children(int32_t b, std::vector<std::array<int32_t, 3>>& out) const {
        const Block& bb = B(b);
        if (bb.t == bb.s) {
            out.push_back({bb.child[0], 0, 0});
            out.push_back({bb.child[1], 1, 0});
            out.push_back({bb.child[2], 1, 1});
        } else {
            for (int k = 0; k < 2; ++k)
                for (int i = 0; i < 2; ++i) out.push_back({bb.child[i + 2 * k], i, k});
        }
    }

    void push_down(int32_t b) {
        Pend pd = std::move(pend[b]);
        pend[b] = Pend();
        if (pd.prods.empty() && pd.pieces.empty()) return;
        std::vector<std::array<int32_t, 3>> ch;
        children(b, ch);
        const Block& bb = B(b);
        for (auto& pr : pd.prods) {
            const int32_t X = pr.first, Y = pr.second;
            const int32_t kx = P.bs[X].kind, ky = P.bs[Y].kind;
            if (kx == ST_SUB && ky == ST_SUB) {
                for (auto& c : ch)
                    for (int j = 0; j < 2; ++j)
                        pend[c[0]].prods.push_back({B(X).child[c[1] + 2 * j], B(Y).child[c[2] + 2 * j]});
            } else if (kx == ST_LR) {
                cur_site = 1;
                Thin Tm = new_thin(bb.s, P.bs[X].cap, P.bs[X].rslot, wnat_of(Y, thin_V(X)));
                hxt(Y, thin_V(X), Tm, 1.0, false);
                pd.pieces.push_back(LPiece{thin_U(X), Tm, -1.0});
                piece_ref(pd.pieces.back(), +1);
            } else if (ky == ST_LR) {
                cur_site = 1;
                Thin Tm = new_thin(bb.t, P.bs[Y].cap, P.bs[Y].rslot, wnat_of(X, thin_V(Y)));
                hxt(X, thin_V(Y), Tm, 1.0, false);
                pd.pieces.push_back(LPiece{Tm, thin_U(Y), -1.0});
                piece_ref(pd.pieces.back(), +1);
            } else {
                throw std::logic_error("push_down: dense factor above the leaf level");
            }
        }
        for (auto& pc : pd.pieces) {
            for (auto& c : ch) {
                const Block& cb = B(c[0]);
                pend[c[0]].pieces.push_back(LPiece{sub(pc.U, cb.t), sub(pc.V, cb.s), pc.alpha});
                piece_ref(pend[c[0]].pieces.back(), +1);
            }
            piece_ref(pc, -1);
        }
    }

    // dense leaf target: t0 holds B; apply pending products and pieces
    // dense leaf target: t0 holds B; apply pending products and pieces.  Long update
    // lists are split: every VM_PARTIAL_TERMS terms form an independent task that
    // accumulates its partial sum into a temporary tile (ring of 64 x 64 slots) as
    // soon as its own operands exist; the target's task then only adds the partials.
    // This moves the bulk of the update off the Cholesky's critical path.
    // The pieces consumed are appended to `rel`: the caller drops their references after
    // emitting the target's program (which may read them).
    void apply_dense_pending(Prog& pg, int32_t b, std::vector<LPiece>& rel) {
        Pend pd = std::move(pend[b]);
        pend[b] = Pend();
        rel.insert(rel.end(), pd.pieces.begin(), pd.pieces.end());
        std::vector<Prog> terms;
        for (auto& pr : pd.prods) {
            const int32_t X = pr.first, Y = pr.second;
            if (P.bs[X].kind != ST_DENSE || P.bs[Y].kind != ST_DENSE)
                throw std::logic_error("leaf product with non-dense factor");
            Prog t;
            ld_dense(t, 1, X);
            ld_dense(t, 2, Y);
            gemm(t, 0, 1, false, 2, true, -1.0, 1.0);
            terms.push_back(std::move(t));
        }
        for (auto& pc : pd.pieces) {
            for (int32_t kc = 0; kc < pc.U.cols; kc += 64) {
                Prog t;
                ld_thin(t, 1, pc.U, pc.U.cluster, kc);
                ld_thin(t, 2, pc.V, pc.V.cluster, kc);
                gemm(t, 0, 1, false, 2, true, pc.alpha, 1.0);
                terms.push_back(std::move(t));
            }
        }
        auto append = [](Prog& dst, const Prog& src) {
            dst.ins.insert(dst.ins.end(), src.ins.begin(), src.ins.end());
            dst.reads.insert(dst.reads.end(), src.reads.begin(), src.reads.end());
            dst.writes.insert(dst.writes.end(), src.writes.begin(), src.writes.end());
        };
        if ((int)terms.size() <= VM_PARTIAL_TERMS) {
            for (auto& t : terms) append(pg, t);
            return;
        }
        const BStore& st = P.bs[b];
        for (size_t c0 = 0; c0 < terms.size(); c0 += VM_PARTIAL_TERMS) {
            Prog pt;
            zero(pt, 0, dstat(st.m), dstat(st.p));
            for (size_t i = c0; i < std::min(terms.size(), c0 + VM_PARTIAL_TERMS); ++i) append(pt, terms[i]);
            const int64_t slot = tmp_alloc(pt.writes);
            VIns sti = mk(VM_ST);
            sti.t0 = 0; sti.rows = dstat(st.m); sti.cols = dstat(st.p); sti.goff = slot; sti.ld = st.m;
            pt.ins.push_back(sti);
            emit_vm(pt);
            VIns ld = mk(VM_LD);
            ld.t0 = 1; ld.rows = dstat(st.m); ld.cols = dstat(st.p); ld.goff = slot; ld.ld = st.m;
            pg.ins.push_back(ld);
            pg.reads.push_back(tmp_res[(slot - P.tmp_off) / TMP_SLOT]);
            op2(pg, VM_ADD, 0, 1);
        }
    }

    // temporary-tile ring for the partial sums (slots of TMP_SLOT doubles; each slot
    // is a dependency resource, so a slot is reused only after its reader ran)
    static constexpr int64_t TMP_SLOT = 64 * 64;
    std::vector<int32_t> tmp_res;
    int64_t tmp_ptr = 0;
    int64_t tmp_alloc(std::vector<int32_t>& writes) {
        const int64_t s = tmp_ptr;
        tmp_ptr = (tmp_ptr + 1) % (int64_t)tmp_res.size();
        writes.push_back(tmp_res[s]);
        return P.tmp_off + s * TMP_SLOT;
    }

    // evaluate product X Y^T into truncation pieces placed at (row0, col0) of the target
    void eval_pieces(int32_t X, int32_t Y, int32_t row0, int32_t col0, std::vector<TPiece>& out,
                     std::vector<std::vector<int32_t>>& pres, std::vector<Thin>& temps) {
        std::vector<int32_t> reads;
        const int32_t kx = P.bs[X].kind, ky = P.bs[Y].kind;
        if (kx == ST_LR) {
            cur_site = 2;
            Thin Tm = new_thin(B(Y).t, P.bs[X].cap, P.bs[X].rslot, wnat_of(Y, thin_V(X)));
            hxt(Y, thin_V(X), Tm, 1.0, false);
            out.push_back(tpiece(thin_U(X), Tm, row0, col0, -1.0, reads));
            pres.push_back(std::move(reads));
            temps.push_back(Tm);
        } else if (ky == ST_LR) {
            cur_site = 2;
            Thin Tm = new_thin(B(X).t, P.bs[Y].cap, P.bs[Y].rslot, wnat_of(X, thin_V(Y)));
            hxt(X, thin_V(Y), Tm, 1.0, false);
            out.push_back(tpiece(Tm, thin_U(Y), row0, col0, -1.0, reads));
            pres.push_back(std::move(reads));
            temps.push_back(Tm);
        } else if (kx == ST_DENSE && ky == ST_DENSE) {
            out.push_back(tpiece(thin_D(X), thin_D(Y), row0, col0, -1.0, reads));
            pres.push_back(std::move(reads));
        } else if (kx == ST_SUB && ky == ST_SUB) {
            const Cluster& rx = C(B(X).t);
            const Cluster& ry = C(B(Y).t);
            for (int i = 0; i < 2; ++i)
                for (int k = 0; k < 2; ++k)
                    for (int j = 0; j < 2; ++j) {
                        const int32_t cx = B(X).child[i + 2 * j], cy = B(Y).child[k + 2 * j];
                        eval_pieces(cx, cy, row0 + (int32_t)(C(B(cx).t).lo - rx.lo),
                                    col0 + (int32_t)(C(B(cy).t).lo - ry.lo), out, pres, temps);
                    }
        } else {
            throw std::logic_error("eval_pieces: mixed dense/subdivided factors");
        }
    }

    TPiece tpiece(const Thin& U, const Thin& V, int32_t row0, int32_t col0, double alpha,
                  std::vector<int32_t>& reads) {
        TPiece p{};
        p.u_off = U.off; p.u_ld = U.ld; p.u_row0 = row0; p.u_rows = (int32_t)C(U.cluster).size();
        p.v_off = V.off; p.v_ld = V.ld; p.v_row0 = col0; p.v_rows = (int32_t)C(V.cluster).size();
        p.w = (U.slot >= 0) ? ddyn(U.cols, U.slot, 0) : dstat(U.cols);
        p.alpha = alpha;
        thin_res(U, reads);
        thin_res(V, reads);
        return p;
    }

    // Where a truncation writes: the block's own factors or a temporary partial sum.
    struct TruncTarget {
        int64_t u_off, v_off;
        int32_t m, q, cap, rslot;
    };
    TruncTarget target_of(int32_t b) const {
        const BStore& s = P.bs[b];
        return TruncTarget{s.u_off, s.v_off, s.m, s.p, s.cap, s.rslot};
    }
    int32_t ready_wave(const std::vector<int32_t>& res) const {
        int32_t w = 0;
        for (int32_t r : res) w = std::max(w, lw_wave[r] + 1);
        return w;
    }

    // low-rank target: gather own + pending and re-truncate once.  A wide sum whose
    // pieces become available at different times is truncated in two steps (split_trunc):
    // the early pieces (and the block's own factors) are merged into a temporary low-rank
    // partial sum as soon as they exist, so the step that waits for the last pieces
    // only handles that partial sum plus those pieces -- a much narrower stack on the
    // Cholesky's critical path.
    void flush_lr(int32_t b, bool force) {
        Pend pd = std::move(pend[b]);
        pend[b] = Pend();
        if (!force && pd.prods.empty() && pd.pieces.empty()) return;
        std::vector<TPiece> pcs;
        std::vector<std::vector<int32_t>> pres;
        std::vector<int32_t> writes;
        std::vector<Thin> temps;
        auto add = [&](const Thin& U, const Thin& V, double alpha) {
            std::vector<int32_t> r;
            pcs.push_back(tpiece(U, V, 0, 0, alpha, r));
            pres.push_back(std::move(r));
        };
        add(thin_U(b), thin_V(b), 1.0);
        for (auto& pc : pd.pieces) add(pc.U, pc.V, pc.alpha);
        for (auto& pr : pd.prods) eval_pieces(pr.first, pr.second, 0, 0, pcs, pres, temps);
        thin_res(thin_U(b), writes);
        thin_res(thin_V(b), writes);
        if (!split_trunc(b, pcs, pres, writes)) {
            std::vector<int32_t> reads;
            for (auto& r : pres) reads.insert(reads.end(), r.begin(), r.end());
            emit_trunc(target_of(b), pcs, reads, writes, 1.0);
        }
        for (auto& pc : pd.pieces) piece_ref(pc, -1);
        for (auto& t : temps) {
            tmp_ref(t, +1);
            tmp_ref(t, -1);
        }
    }

    bool split_trunc(int32_t b, const std::vector<TPiece>& pcs, const std::vector<std::vector<int32_t>>& pres,
                     std::vector<int32_t>& writes) {
        const BStore& s = P.bs[b];
        const int32_t n = (int32_t)pcs.size();
        int32_t ktot = 0;
        for (auto& p : pcs) ktot += p.w.stat;
        if (!split_enabled || n < 4 || ktot <= 4 * s.cap || trunc_exact_path(s.m, s.p, ktot)) return false;
        std::vector<int32_t> wv(n), order;
        for (int32_t i = 0; i < n; ++i) wv[i] = ready_wave(pres[i]);
        for (int32_t i = 1; i < n; ++i) order.push_back(i);   // the block's own factors are early by nature
        std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t c) { return wv[a] > wv[c]; });
        std::vector<char> late(n, 0);
        int32_t klate = 0;
        for (int32_t i : order) {
            if (klate > 0 && klate + pcs[i].w.stat > 2 * s.cap) break;
            late[i] = 1;
            klate += pcs[i].w.stat;
        }
        int32_t kearly = ktot - klate, wearly = 0, wlate = 0;
        for (int32_t i = 0; i < n; ++i) {
            if (late[i]) wlate = std::max(wlate, wv[i]);
            else wearly = std::max(wearly, wv[i]);
        }
        if (kearly <= 2 * s.cap || wearly >= wlate) return false;   // nothing to hide
        // partial sum of the early pieces into a temporary (arena) low-rank pair, rank slot of its own
        const int32_t cap_t = std::min(std::min(s.m, s.p), std::min(2 * s.cap, TR_LMAX - TR_RB));
        const int32_t slot_t = P.n_slots++;
        Thin Ut = new_thin(B(b).t, cap_t, slot_t, wearly);
        Thin Vt = new_thin(B(b).s, cap_t, slot_t, wearly);
        tmp_ref(Ut, +1);
        tmp_ref(Vt, +1);
        std::vector<TPiece> pe;
        std::vector<int32_t> re, we;
        for (int32_t i = 0; i < n; ++i)
            if (!late[i]) {
                pe.push_back(pcs[i]);
                re.insert(re.end(), pres[i].begin(), pres[i].end());
            }
        thin_res(Ut, we);
        thin_res(Vt, we);
        emit_trunc(TruncTarget{Ut.off, Vt.off, s.m, s.p, cap_t, slot_t}, pe, re, we, TRUNC_SPLIT_SHARE);
        // final step: partial sum + the late pieces -> the block
        std::vector<TPiece> pf;
        std::vector<int32_t> rf;
        pf.push_back(tpiece(Ut, Vt, 0, 0, 1.0, rf));
        for (int32_t i = 0; i < n; ++i)
            if (late[i]) {
                pf.push_back(pcs[i]);
                rf.insert(rf.end(), pres[i].begin(), pres[i].end());
            }
        emit_trunc(target_of(b), pf, rf, writes, 1.0 - TRUNC_SPLIT_SHARE);
        tmp_ref(Ut, -1);
        tmp_ref(Vt, -1);
        ++n_split;
        return true;
    }
    static constexpr double TRUNC_SPLIT_SHARE = 0.25;   // accuracy share of the partial merge
    // Off by default (HM_TRUNC_SPLIT=1 enables it): measured at n = 64k it LOSES -- one
    // evaluation 422 -> 560 ms, 4 co-scheduled 4.68 -> 3.76 evals/s -- the partial merge
    // is rarely off the critical path in the executor's actual order (the wave proxy
    // is too coarse) and the extra truncations add work.
    bool split_enabled = false;
    int64_t n_split = 0;

    void emit_trunc(const TruncTarget& tg, const std::vector<TPiece>& pcs, std::vector<int32_t>& reads,
                    std::vector<int32_t>& writes, double eps_scale) {
        std::sort(reads.begin(), reads.end());
        reads.erase(std::unique(reads.begin(), reads.end()), reads.end());
        int32_t kt = 0, wmax = 0;
        for (auto& p : pcs) {
            kt += p.w.stat;
            wmax = std::max(wmax, p.w.stat);
        }
        const int32_t nsub = trunc_nsub(tg.m, tg.q, kt, coop_max);
        const int64_t wsz = trunc_ws_size(tg.m, tg.q, tg.cap, kt, nsub);
        const int64_t nch = (wsz + ring_chunk - 1) / ring_chunk;
        if (4 * nch > ring_nchunks) grow_ring(4 * nch);   // keep >= 4 workspaces of this size in flight
        if (ring_ptr + nch > ring_nchunks) ring_ptr = 0;
        const int64_t ws_off = ring_ptr * ring_chunk;    // relative to the ring; rebased after planning
        for (int64_t c = 0; c < nch; ++c) writes.push_back(ring_res[ring_ptr + c]);
        ring_ptr += nch;
        std::vector<int32_t> deps;
        int32_t w = wave_of(reads, writes, deps);
        TTask t{};
        t.u_out = tg.u_off; t.v_out = tg.v_off;
        t.m = tg.m; t.q = tg.q; t.cap = tg.cap; t.rslot = tg.rslot;
        t.piece_begin = (int32_t)ph->tp.size();
        t.piece_count = (int32_t)pcs.size();
        t.kmax_tot = kt;
        t.wmax = wmax;
        t.ws_size = wsz;
        t.ws = ws_off;
        t.eps_scale = eps_scale;
        if ((int32_t)pcs.size() > TR_PMAX) throw std::logic_error("truncation with more than TR_PMAX pieces");
        t.nsub = nsub;
        t.bar = 0;
        if (t.nsub > 1) {                                 // two counters: the group, then its shrunk core
            t.bar = ph->n_bars;
            ph->n_bars += 2;
        }
        ph->tp.insert(ph->tp.end(), pcs.begin(), pcs.end());
        xraw.push_back({w, 1, (int32_t)traw.size(), std::move(deps)});
        traw.push_back({w, t});
        ++n_tasks;
    }

    // ---- H-Cholesky recursion -----------------------------------------------
    void chol(int32_t t) {
        const int32_t d = P.diag_of[t];
        if (P.bs[d].kind == ST_SUB) {
            push_down(d);
            const int32_t t0 = C(t).child[0], t1 = C(t).child[1];
            chol(t0);
            const int32_t off = B(d).child[1];   // (t1, t0)
            trsm(off);
            pend[B(d).child[2]].prods.push_back({off, off});
            chol(t1);
            if (P.bs[off].x_off >= 0) {
                // X10 = -L11^{-1} L10 L00^{-1} for one-task forward solves over t (fsolve)
                const BStore& so = P.bs[off];
                Prog pg;
                ld_inv(pg, 0, P.diag_of[t1]);
                ld_dense(pg, 1, off);
                gemm(pg, 2, 0, false, 1, false, 1.0, 0.0);
                ld_inv(pg, 0, P.diag_of[t0]);
                gemm(pg, 1, 2, false, 0, false, -1.0, 0.0);
                VIns st = mk(VM_ST);
                st.t0 = 1; st.rows = dstat(so.m); st.cols = dstat(so.p); st.goff = so.x_off; st.ld = so.m;
                pg.ins.push_back(st);
                pg.writes.push_back(so.x_res);
                emit_vm(pg);
            }
        } else {
            Prog pg;
            std::vector<LPiece> rel;
            ld_dense(pg, 0, d);
            apply_dense_pending(pg, d, rel);
            const int32_t li = P.leaf_begin[t];
            op2(pg, VM_POTRF, 0, 0, P.logd_off + li);
            st_dense(pg, 0, d);
            op2(pg, VM_TRTRI, 1, 0);                     // L^{-1} for the block row's TRSMs / solves
            {
                const BStore& sd = P.bs[d];
                VIns st = mk(VM_ST);
                st.t0 = 1; st.rows = dstat(sd.m); st.cols = dstat(sd.m); st.goff = sd.inv_off; st.ld = sd.m;
                pg.ins.push_back(st);
                pg.writes.push_back(sd.inv_res);
            }
            emit_vm(pg);
            for (auto& pc : rel) piece_ref(pc, -1);
        }
    }

    void trsm(int32_t b) {
        const Block& bb = B(b);
        const int32_t s = bb.s;
        const BStore& st = P.bs[b];
        if (st.kind == ST_SUB) {
            push_down(b);
            const int32_t ds = P.diag_of[s];
            for (int i = 0; i < 2; ++i) trsm(bb.child[i]);                     // (r_i, s0)
            for (int i = 0; i < 2; ++i) pend[bb.child[i + 2]].prods.push_back({bb.child[i], B(ds).child[1]});
            for (int i = 0; i < 2; ++i) trsm(bb.child[i + 2]);                 // (r_i, s1)
        } else if (st.kind == ST_DENSE) {
            Prog pg;
            std::vector<LPiece> rel;
            ld_dense(pg, 0, b);
            apply_dense_pending(pg, b, rel);
            ld_inv(pg, 1, P.diag_of[s]);                // B <- B L^{-T} = B (L^{-1})^T
            gemm(pg, 2, 0, false, 1, true, 1.0, 0.0);
            st_dense(pg, 2, b);
            emit_vm(pg);
            for (auto& pc : rel) piece_ref(pc, -1);
        } else {
            flush_lr(b, false);
            fsolve(s, thin_V(b));
        }
    }

    // ---- phase bookkeeping -------------------------------------------------
    void begin_phase(Phase& p) {
        ph = &p;
        p.n_bars = 0;
        vraw.clear();
        traw.clear();
        xraw.clear();
        ring_ptr = 0;
        tmp_ptr = 0;
        arena_new_phase();
        std::fill(lw_wave.begin(), lw_wave.end(), -1);
        std::fill(rd_wave.begin(), rd_wave.end(), -1);
        std::fill(lw_task.begin(), lw_task.end(), -1);
        for (auto& v : rd_tasks) v.clear();
    }
    void end_phase() {
        int32_t nw = 0;
        for (auto& v : xraw) nw = std::max(nw, v.wave + 1);
        // stable order by wave of the VM / truncation lists (local -> sorted position)
        auto sorted_pos = [](const auto& raw) {
            std::vector<int32_t> idx(raw.size()), pos(raw.size());
            for (size_t i = 0; i < raw.size(); ++i) idx[i] = (int32_t)i;
            std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return raw[a].first < raw[b].first; });
            for (size_t i = 0; i < idx.size(); ++i) pos[idx[i]] = (int32_t)i;
            return std::make_pair(idx, pos);
        };
        auto [vidx, vpos] = sorted_pos(vraw);
        auto [tidx, tpos] = sorted_pos(traw);
        ph->nwaves = nw;
        ph->v_wave_begin.assign(nw + 1, 0);
        ph->t_wave_begin.assign(nw + 1, 0);
        ph->vt.clear();
        ph->tt.clear();
        {
            size_t k = 0;
            for (int32_t w = 0; w < nw; ++w) {
                ph->v_wave_begin[w] = (int32_t)k;
                while (k < vidx.size() && vraw[vidx[k]].first == w) ph->vt.push_back(vraw[vidx[k++]].second);
            }
            ph->v_wave_begin[nw] = (int32_t)k;
        }
        {
            size_t k = 0;
            for (int32_t w = 0; w < nw; ++w) {
                ph->t_wave_begin[w] = (int32_t)k;
                while (k < tidx.size() && traw[tidx[k]].first == w) ph->tt.push_back(traw[tidx[k++]].second);
            }
            ph->t_wave_begin[nw] = (int32_t)k;
        }
        // unified topological list for the persistent executor
        std::vector<int32_t> xidx(xraw.size()), xpos(xraw.size());
        for (size_t i = 0; i < xraw.size(); ++i) xidx[i] = (int32_t)i;
        std::stable_sort(xidx.begin(), xidx.end(), [&](int32_t a, int32_t b) { return xraw[a].wave < xraw[b].wave; });
        for (size_t i = 0; i < xidx.size(); ++i) xpos[xidx[i]] = (int32_t)i;
        // a cooperative truncation occupies nsub consecutive entries (leader first);
        // its successors wait on the leader, which publishes after the group's last barrier
        std::vector<int32_t> xlead(xraw.size());
        {
            int32_t pos = 0;
            for (size_t i = 0; i < xidx.size(); ++i) {
                const XRaw& r = xraw[xidx[i]];
                xlead[xidx[i]] = pos;
                pos += (r.kind == 1) ? ph->tt[tpos[r.local]].nsub : 1;
            }
        }
        ph->xt.clear();
        ph->xdeps.clear();
        for (size_t i = 0; i < xidx.size(); ++i) {
            const XRaw& r = xraw[xidx[i]];
            XTask x{};
            x.kind = r.kind;
            x.idx = r.kind == 0 ? vpos[r.local] : tpos[r.local];
            x.dep_begin = (int32_t)ph->xdeps.size();
            const int32_t me = xlead[xidx[i]];
            for (int32_t d : r.deps) {
                if (xlead[d] >= me) throw std::logic_error("planner: dependency not in topological order");
                ph->xdeps.push_back(xlead[d]);
            }
            x.dep_count = (int32_t)ph->xdeps.size() - x.dep_begin;
            x.nsub = (r.kind == 1) ? ph->tt[x.idx].nsub : 1;
            for (int32_t sb = 0; sb < x.nsub; ++sb) {
                x.sub = sb;
                ph->xt.push_back(x);
            }
        }
        ph = nullptr;
    }
};

}  // namespace

std::string Plan::summary() const {
    char buf[512];
    std::snprintf(buf, sizeof(buf),
                  "blocks=%zu leaves=%d slots=%d pool_blocks=%.3f GB pool_total=%.3f GB | chol: %zu vm + %zu trunc "
                  "tasks, %d waves, %lld launches | solve: %zu tasks, %d waves",
                  bs.size(), n_leaves, n_slots, pool_blocks * 8e-9, pool_total * 8e-9, chol.vt.size(), chol.tt.size(),
                  chol.nwaves, (long long)chol.n_launches(), solve.vt.size() + solve.tt.size(), solve.nwaves);
    return buf;
}

void build_plan(const Tree& T0, int32_t kmax, Plan& P, int32_t coop_max, int64_t arena_budget,
                const std::vector<int32_t>* cap_hint, bool assembly_only) {
    // mixed-depth leaves (n / 2^l straddling n_min) and leaves above one 64 x 64 tile
    // (n_min up to 128) are planned on the refined storage tree (tree.h refine_for_plan):
    // same C~, dense blocks split into equal-depth tile-sized sub-blocks
    Tree Tr;
    const bool ready = plan_ready(T0, TILE_MAX_LEAF);
    if (!ready) refine_for_plan(T0, TILE_MAX_LEAF, Tr);
    const Tree& T = ready ? T0 : Tr;
    P = Plan();
    P.kmax = kmax;
    const int32_t nc = (int32_t)T.clusters.size();
    // leaves in tree order and per-cluster leaf ranges
    P.leaf_begin.assign(nc, 0);
    P.leaf_count.assign(nc, 0);
    {
        // pre-order == storage order; leaves appear in index order, all at one depth (plan_ready)
        for (int32_t c = 0; c < nc; ++c)
            if (T.clusters[c].leaf()) P.leaf_cluster.push_back(c);
        P.n_leaves = (int32_t)P.leaf_cluster.size();
        // leaf_begin via post-order accumulation (children after parents in pre-order: iterate backwards)
        std::vector<int32_t> first(nc, INT32_MAX);
        for (int32_t i = 0; i < P.n_leaves; ++i) {
            first[P.leaf_cluster[i]] = i;
            P.leaf_count[P.leaf_cluster[i]] = 1;
        }
        for (int32_t c = nc - 1; c >= 0; --c) {
            const Cluster& cl = T.clusters[c];
            if (!cl.leaf()) {
                first[c] = std::min(first[cl.child[0]], first[cl.child[1]]);
                P.leaf_count[c] = P.leaf_count[cl.child[0]] + P.leaf_count[cl.child[1]];
            }
        }
        for (int32_t c = 0; c < nc; ++c) P.leaf_begin[c] = first[c];
    }
    Builder bld(T, P);
    if (coop_max < 1 || coop_max > TR_COOP_MAX) throw std::invalid_argument("coop_max must be in [1, 32]");
    bld.coop_max = coop_max;
    // block storage
    const int32_t nb = (int32_t)T.blocks.size();
    P.bs.assign(nb, BStore());
    P.diag_of.assign(nc, -1);
    for (int32_t b = 0; b < nb; ++b) {
        const Block& bk = T.blocks[b];
        if (bk.t == bk.s) P.diag_of[bk.t] = b;
        BStore& s = P.bs[b];
        const Cluster& ct = T.clusters[bk.t];
        const Cluster& cs = T.clusters[bk.s];
        s.m = (int32_t)ct.size();
        s.p = (int32_t)cs.size();
        const bool leafpair = ct.leaf() && cs.leaf();
        if (bk.kind == BK_SUB) {
            s.kind = ST_SUB;
        } else if (bk.kind == BK_DENSE || leafpair) {
            s.kind = ST_DENSE;
            s.d_off = bld.alloc((int64_t)s.m * s.p);
            s.d_res = bld.new_res(1);
            P.bytes_C += 8LL * s.m * s.p;
            if (bk.t == bk.s) {
                s.inv_off = bld.alloc((int64_t)s.m * s.m);
                s.inv_res = bld.new_res(1);
            }
        } else {
            s.kind = ST_LR;
            s.cap = std::min(kmax, std::min(s.m, s.p));
            if (cap_hint && b < (int32_t)cap_hint->size() && (*cap_hint)[b] > 0) s.cap = std::min(s.cap, (*cap_hint)[b]);
            s.rslot = P.n_slots++;
            s.u_off = bld.alloc((int64_t)s.m * s.cap);
            s.v_off = bld.alloc((int64_t)s.p * s.cap);
            s.u_res0 = bld.new_res(P.leaf_count[bk.t]);
            s.v_res0 = bld.new_res(P.leaf_count[bk.s]);
            P.bytes_C += 8LL * (s.m + s.p) * s.cap;
        }
    }
    // X10 blocks of the two-leaf diagonal clusters (see BStore::x_off)
    for (int32_t c = 0; c < nc; ++c) {
        const Cluster& cl = T.clusters[c];
        if (cl.leaf() || !T.clusters[cl.child[0]].leaf() || !T.clusters[cl.child[1]].leaf()) continue;
        const int32_t d = P.diag_of[c];
        if (d < 0 || P.bs[d].kind != ST_SUB) continue;
        BStore& o = P.bs[T.blocks[d].child[1]];
        if (o.kind != ST_DENSE) continue;
        o.x_off = bld.alloc((int64_t)o.m * o.p);
        o.x_res = bld.new_res(1);
    }
    P.logd_off = bld.alloc(P.n_leaves);
    P.zw = 64;
    P.z_off = bld.alloc((int64_t)T.n * P.zw);
    P.z_slot = P.n_slots++;
    P.n_block_slots = P.n_slots;
    const int32_t z_res0 = bld.new_res(P.n_leaves);
    P.pool_blocks = bld.bump;
    // temporary 64 x 64 tiles for split dense updates (see apply_dense_pending)
    {
        const int64_t nslots = 8192;   // 256 MiB
        P.tmp_off = bld.alloc(nslots * Builder::TMP_SLOT);
        for (int64_t i = 0; i < nslots; ++i) bld.tmp_res.push_back(bld.new_res(1));
    }
    // truncation workspace ring: starts at >= 4x the largest recompression workspace and,
    // within 1 GiB, at the sum of all of them (the recompressions are independent: ring
    // reuse is their only dependency, so a small ring would chain them); grows to >= 4x
    // the largest workspace the Cholesky emits
    std::vector<int32_t> lr_order;
    {
        int64_t maxs = 0, sum = 0;
        for (int32_t b = 0; b < nb; ++b) {
            const BStore& s = P.bs[b];
            if (s.kind != ST_LR) continue;
            lr_order.push_back(b);
            const int64_t w = trunc_ws_size(s.m, s.p, s.cap, s.cap, trunc_nsub(s.m, s.p, s.cap, coop_max));
            maxs = std::max(maxs, w);
            sum += w;
            maxs = std::max(maxs, trunc_ws_size(s.m, s.p, s.cap, TR_EXACT_K + 1, 1));
        }
        bld.ring_chunk = int64_t(1) << 16;   // 512 KiB
        const int64_t want = std::max<int64_t>(4 * maxs, std::min<int64_t>(int64_t(1) << 27, sum + sum / 8));
        bld.grow_ring((want + bld.ring_chunk - 1) / bld.ring_chunk);
        // largest first: the long recompressions start at once and the ring wraps onto short ones
        std::stable_sort(lr_order.begin(), lr_order.end(), [&](int32_t a, int32_t b) {
            return (int64_t)P.bs[a].m + P.bs[a].p > (int64_t)P.bs[b].m + P.bs[b].p;
        });
    }
    // assembly tasks
    for (int32_t b = 0; b < nb; ++b) {
        const Block& bk = T.blocks[b];
        const BStore& s = P.bs[b];
        const Cluster& ct = T.clusters[bk.t];
        const Cluster& cs = T.clusters[bk.s];
        if (s.kind == ST_DENSE) {
            P.dgen.push_back(DenseGenTask{s.d_off, (int32_t)ct.lo, (int32_t)cs.lo, s.m, s.p});
        } else if (s.kind == ST_LR) {
            P.aca.push_back(AcaTask{s.u_off, s.v_off, (int32_t)ct.lo, (int32_t)cs.lo, s.m, s.p, s.cap, s.rslot});
        }
    }
    // largest ACA blocks first: one CTA per block, so the long ones must not start last
    std::stable_sort(P.aca.begin(), P.aca.end(),
                     [](const AcaTask& a, const AcaTask& b) { return (int64_t)a.m + a.q > (int64_t)b.m + b.q; });
    bld.pend.assign(nb, Pend());
    // temporaries of every phase live in one arena above the permanent storage
    bld.arena_base = bld.bump;
    if (const char* am = std::getenv("HM_ARENA_MODE")) bld.arena_mode = std::atoi(am);
    if (const char* wm = std::getenv("HM_WNAT_MODE")) bld.wnat_mode = std::atoi(wm);
    if (const char* sp = std::getenv("HM_TRUNC_SPLIT")) bld.split_enabled = std::atoi(sp) != 0;
    bld.arena_budget = arena_budget;
    if (const char* ab = std::getenv("HM_ARENA_BUDGET")) bld.arena_budget = std::atoll(ab);
    // recompression of every ACA block: a truncation with the block itself as the only piece
    bld.begin_phase(P.recompress);
    for (int32_t b : lr_order) bld.flush_lr(b, true);
    bld.end_phase();
    if (!assembly_only) {   // (assembly-only plans: rank probes of hm_build's adaptive capacities)
        // H-Cholesky
        bld.begin_phase(P.chol);
        bld.n_tasks = 0;
        bld.chol(0);
        P.n_tasks_chol = bld.n_tasks;
        bld.end_phase();
        for (auto& pd : bld.pend)
            if (!pd.prods.empty() || !pd.pieces.empty()) throw std::logic_error("planner: unapplied pending update");
        // forward solve and sampler on the z buffer (rows = root cluster, tree order)
        Thin Z;
        Z.off = P.z_off; Z.ld = (int32_t)T.n; Z.cluster = 0; Z.cols = P.zw; Z.slot = P.z_slot; Z.res0 = z_res0;
        bld.begin_phase(P.solve);
        bld.fsolve(0, Z);
        bld.end_phase();
        bld.begin_phase(P.lmul);
        bld.lmul(0, Z);
        bld.end_phase();
    }
    for (const auto& a : bld.tmps)
        if (a.refs != 0) throw std::logic_error("planner: live temporary at the end of planning");
    P.n_split = bld.n_split;
    P.arena_off = bld.arena_base;
    P.arena_size = bld.arena_top;
    bld.bump = bld.arena_base + bld.arena_top;
    // place the ring and rebase every truncation workspace offset onto it
    P.ring_size = bld.ring_nchunks * bld.ring_chunk;
    P.ring_off = bld.alloc(P.ring_size);
    for (Phase* ph : {&P.recompress, &P.chol, &P.solve, &P.lmul})
        for (TTask& t : ph->tt) t.ws += P.ring_off;
    P.pool_total = bld.bump;
    if (std::getenv("HM_PLAN_VERBOSE"))
        std::fprintf(stderr, "plan: blocks(C~ at capacity)=%.3f GB z=%.3f GB tmp=%.3f GB ring=%.3f GB arena=%.3f GB total=%.3f GB\n",
                     8e-9 * P.bytes_C / 8, 8e-9 * (double)T.n * P.zw, 8e-9 * 8192 * 4096.0, 8e-9 * P.ring_size,
                     8e-9 * P.arena_size, 8e-9 * P.pool_total);
    if (std::getenv("HM_PLAN_VERBOSE"))
        std::fprintf(stderr, "temporaries allocated: push_down %.3f GB, eval_pieces %.3f GB, cores %.3f GB\n",
                     1e-9 * bld.site_bytes[1], 1e-9 * bld.site_bytes[2], 1e-9 * bld.site_bytes[3]);
}

}  // namespace hm

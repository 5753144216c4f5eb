// H-matrix entry points of include/hmlik.h: hm_build, hm_assemble, hm_cholesky,
// hm_loglik, hm_loglik_batch, hm_sample, hm_stats, hm_timings.
//
// The handle owns: the host tree + plan (built once per location set), one
// device pool holding every block of C~ / L~ plus all planned temporaries,
// the device copies of the task lists, and a CUDA stream.  Each phase is a
// sequence of waves; a wave launches the tile VM for its VM tasks and the
// truncation kernel for its truncation tasks.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <memory>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include "../../include/hmlik.h"
#include "api_util.h"
#include "common.h"
#include "hm_kernels.h"
#include "plan.h"
#include "sched.h"
#include "tree.h"

namespace hm {

enum KFamily { KF_DGEN = 0, KF_ACA = 1, KF_TRUNC = 2, KF_VM = 3, KF_AUX = 4, KF_EXEC = 5, KF_N = 6 };

struct DPhase {
    DevBuf ins, vt, tt, tp, xt, xd, terms;
    DevBuf xr, su2, qbase, slot_init, ctl_init;   // xr: xt with (dep_begin, dep_count) := successor range
    int max_nsub = 1;   // ready-queue schedule (sched.h)
    const Phase* ph = nullptr;
};

}  // namespace hm

using namespace hm;

struct hm_handle_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    Tree T;
    Plan P;
    hm_params prm{};
    hm_theta theta{};
    MaternParams mp{};
    DevBuf pool, pts, perm, ranks, flags, out, zio, dgen, aca, ctr;
    // persistent executor state: completion flags (== epoch when done) and claim counter
    DevBuf done, counter, bars;
    DevBuf rq_cnt, rq_slot, rq_ctl;   // ready-queue executor: arrival counters, queue slots, {head, tail} + finished
    int epoch = 0;
    int exec_grid_cap = 0;   // > 0: at most this many executor CTAs (co-scheduled handles, hm_set_exec_grid)
    int exec_mode = 2;   // 2 = persistent ready-queue executor, 1 = persistent topological-claim executor,
                         // 0 = one launch per wave
    DevBuf trace;        // per-task timestamps of the last executor launch (hm_trace)
    bool tracing = false;
    bool poison = false;
    bool abs_eps = true;   // block accuracy eps absolute (x sigma^2, default) or relative (rel_eps)
    double eps_k = 0.0;    // eps as the kernels see it: > 0 relative, < 0 absolute (assembly, recompression)
    double eps_kc = 0.0;   // the same for the truncations of the H-Cholesky (hm_params.eps_chol)
    double eps_run = 0.0;  // the value run_phase passes to the kernels (set per phase)
    int64_t trace_n = 0;
    // profiling: per kernel family (KF_*) launch counts (always) and, when
    // enabled, a CUDA event pair around every launch on the handle's stream
    bool profiling = false;
    int64_t launches[KF_N] = {0, 0, 0, 0, 0, 0};
    std::vector<cudaEvent_t> evpool;
    std::vector<std::pair<int, int>> evlog;   // (family, index of first event of the pair)
    DPhase rec, chol, solve, lmul;
    bool assembled = false, factored = false;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    double ms[3] = {0, 0, 0};
    int max_rank_C = 0, max_rank_L = 0;
    std::vector<int> h_ranks;
    // pinned host staging for host-buffer calls (pageable copies would serialise
    // co-scheduled handles' streams)
    double* pin_z = nullptr;
    size_t pin_z_n = 0;
    double* pin_out = nullptr;
    size_t pin_out_n = 0;
    // hm_loglik_batch: S - 1 sibling executors on the same tree + plan (own pool, stream)
    std::vector<std::unique_ptr<hm_handle_s>> subs;
    int batch_streams = 0;   // 0 = auto (hm_set_batch_streams)
    std::vector<int32_t> cap_hint;   // adaptive rank capacities per plan block (hm_params.adaptive_cap)
    int cap_retries = 0;
    ~hm_handle_s() {
        if (pin_z) cudaFreeHost(pin_z);
        if (pin_out) cudaFreeHost(pin_out);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : evpool)
            if (e) cudaEventDestroy(e);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }
};

namespace {

template <class T>
void upload(DevBuf& b, const std::vector<T>& v, cudaStream_t st) {
    b.alloc(sizeof(T) * (v.size() + 1));
    if (!v.empty()) HM_CUDA_TRY(cudaMemcpyAsync(b.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
}

void upload_phase(DPhase& d, const Phase& p, cudaStream_t st) {
    upload(d.ins, p.ins, st);
    upload(d.vt, p.vt, st);
    upload(d.tt, p.tt, st);
    upload(d.tp, p.tp, st);
    upload(d.xt, p.xt, st);
    upload(d.terms, p.terms, st);
    upload(d.xd, p.xdeps, st);
    Sched sc;
    build_sched(p, sc);
    {
        std::vector<XTask> xr(p.xt);
        for (size_t i = 0; i < xr.size(); ++i) {
            xr[i].dep_begin = sc.succ_begin[i];
            xr[i].dep_count = sc.succ_begin[i + 1] - sc.succ_begin[i];
        }
        upload(d.xr, xr, st);
        HM_CUDA_TRY(cudaStreamSynchronize(st));
    }
    upload(d.su2, sc.succ2, st);
    d.max_nsub = sc.max_nsub;
    upload(d.qbase, sc.qbase, st);
    upload(d.slot_init, sc.slot_init, st);
    upload(d.ctl_init, sc.ctl_init, st);
    HM_CUDA_TRY(cudaStreamSynchronize(st));   // sc's host vectors die here
    d.ph = &p;
}

// Profiling bracket around one launch of kernel family f.
struct Launch {
    hm_handle_s* h;
    int f;
    int idx = -1;
    Launch(hm_handle_s* hh, int fam) : h(hh), f(fam) {
        ++h->launches[f];
        if (!h->profiling) return;
        idx = (int)(2 * h->evlog.size());
        while ((int)h->evpool.size() < idx + 2) {
            cudaEvent_t e;
            HM_CUDA_TRY(cudaEventCreate(&e));
            h->evpool.push_back(e);
        }
        HM_CUDA_TRY(cudaEventRecord(h->evpool[idx], h->stream));
    }
    ~Launch() {
        if (idx < 0) return;
        cudaEventRecord(h->evpool[idx + 1], h->stream);
        h->evlog.push_back({f, idx});
    }
};

void plan_to_fit(hm_handle_s* h);
void setup_device(hm_handle_s* h);

void run_phase(hm_handle_s* h, const DPhase& d) {
    const Phase& p = *d.ph;
    if (h->poison)   // diagnostics (HM_POISON_RING=1): NaN-fill the truncation workspaces first
        HM_CUDA_TRY(cudaMemsetAsync(h->pool.as<double>() + h->P.ring_off, 0xFF, sizeof(double) * h->P.ring_size, h->stream));
    double* pool = h->pool.as<double>();
    int* ranks = h->ranks.as<int>();
    int* flags = h->flags.as<int>();
    double* ctr = h->ctr.as<double>();
    if (h->exec_mode == 2) {
        Launch L(h, KF_EXEC);
        if (h->tracing)
            HM_CUDA_TRY(cudaMemsetAsync((char*)h->trace.p + 32 * p.xt.size(), 0, 8 * 64 * p.xt.size(), h->stream));
        launch_exec_rq(d.xr.as<XTask>(), (int)p.xt.size(), d.su2.as<int32_t>(), d.qbase.as<int32_t>(), d.slot_init.as<int32_t>(), d.ctl_init.as<int32_t>(),
                       h->rq_cnt.as<int>(), h->rq_slot.as<int>(), h->rq_ctl.as<int>(), d.vt.as<VTask>(),
                       d.ins.as<VIns>(), d.terms.as<VTerm>(), d.tt.as<TTask>(), d.tp.as<TPiece>(), pool, ranks, flags,
                       ctr, h->eps_run, h->tracing ? (unsigned long long*)h->trace.p : nullptr, h->bars.as<int>(),
                       p.n_bars, d.max_nsub, h->exec_grid_cap, h->stream);
        if (h->tracing) h->trace_n = (int64_t)p.xt.size();
        HM_CUDA_TRY(cudaGetLastError());
        return;
    }
    if (h->exec_mode == 1) {
        Launch L(h, KF_EXEC);
        ++h->epoch;
        if (h->tracing)
            HM_CUDA_TRY(cudaMemsetAsync((char*)h->trace.p + 32 * p.xt.size(), 0, 8 * 64 * p.xt.size(), h->stream));
        launch_exec(d.xt.as<XTask>(), (int)p.xt.size(), d.xd.as<int32_t>(), d.vt.as<VTask>(), d.ins.as<VIns>(),
                    d.terms.as<VTerm>(), d.tt.as<TTask>(), d.tp.as<TPiece>(), pool, ranks, flags, ctr, h->eps_run, h->done.as<int>(),
                    h->counter.as<int>(), h->epoch,
                    h->tracing ? (unsigned long long*)h->trace.p : nullptr, h->bars.as<int>(), p.n_bars, h->stream);
        if (h->tracing) h->trace_n = (int64_t)p.xt.size();
        HM_CUDA_TRY(cudaGetLastError());
        return;
    }
    for (int w = 0; w < p.nwaves; ++w) {
        const int v0 = p.v_wave_begin[w], v1 = p.v_wave_begin[w + 1];
        const int t0 = p.t_wave_begin[w], t1 = p.t_wave_begin[w + 1];
        if (t1 > t0) {
            Launch L(h, KF_TRUNC);
            launch_trunc(d.tt.as<TTask>() + t0, t1 - t0, d.tp.as<TPiece>(), pool, ranks, flags, h->eps_run, ctr,
                         h->stream);
        }
        if (v1 > v0) {
            Launch L(h, KF_VM);
            launch_vm(d.vt.as<VTask>() + v0, v1 - v0, d.ins.as<VIns>(), d.terms.as<VTerm>(), pool, ranks, flags, ctr,
                      h->stream);
        }
    }
    HM_CUDA_TRY(cudaGetLastError());
}

float elapsed(hm_handle_s* h) {
    float t = 0;
    HM_CUDA_TRY(cudaEventElapsedTime(&t, h->ev[0], h->ev[1]));
    return t;
}

void read_flags(hm_handle_s* h, int f[4]) {
    HM_CUDA_TRY(cudaMemcpyAsync(f, h->flags.p, sizeof(int) * 4, cudaMemcpyDeviceToHost, h->stream));
    HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
}

int max_rank(hm_handle_s* h) {
    h->h_ranks.resize(h->P.n_slots);
    if (h->P.n_slots == 0) return 0;
    HM_CUDA_TRY(cudaMemcpyAsync(h->h_ranks.data(), h->ranks.p, sizeof(int) * h->P.n_slots, cudaMemcpyDeviceToHost,
                                h->stream));
    HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    int mx = 0;
    for (int i = 0; i < h->P.n_block_slots; ++i)   // blocks only: z_slot is the RHS width, later
        if (i != h->P.z_slot) mx = std::max(mx, h->h_ranks[i]);   // slots hold split truncations' partial sums
    return mx;
}

// grow adaptive capacities after an overflow and re-plan (the handle keeps theta)
void regrow_caps(hm_handle_s* h) {
    ++h->cap_retries;
    for (auto& c : h->cap_hint)
        if (c > 0) c = std::min(h->prm.kmax, (2 * c + 3) & ~3);
    h->pool.release();
    plan_to_fit(h);
    setup_device(h);
}

// aca_ranks (rank probe): receives every slot's rank after ACA, before the recompression
void do_assemble(hm_handle_s* h, hm_theta th, std::vector<int>* aca_ranks = nullptr) {
    check_theta(th);
    h->theta = th;
    h->eps_k = h->abs_eps ? -h->prm.eps * th.sigma2 : h->prm.eps;
    h->eps_kc = h->abs_eps ? -h->prm.eps_chol * th.sigma2 : h->prm.eps_chol;
    h->eps_run = h->eps_k;
    matern_setup(th.sigma2, th.ell, th.nu, h->mp);
    HM_CUDA_TRY(cudaMemsetAsync(h->flags.p, 0, sizeof(int) * 4, h->stream));
    HM_CUDA_TRY(cudaEventRecord(h->ev[0], h->stream));
    {
        Launch L(h, KF_DGEN);
        launch_dense_gen(h->dgen.as<DenseGenTask>(), (int)h->P.dgen.size(), h->pts.as<double>(),
                         h->pool.as<double>(), h->mp, h->ctr.as<double>(), h->stream);
    }
    // ACA at eps/4, then recompression to eps (QR + SVD)
    {
        Launch L(h, KF_ACA);
        launch_aca(h->aca.as<AcaTask>(), (int)h->P.aca.size(), h->pts.as<double>(), h->pool.as<double>(),
                   h->ranks.as<int>(), h->flags.as<int>(), h->mp, 0.25 * h->eps_k, h->ctr.as<double>(), h->stream);
    }
    if (aca_ranks) {
        aca_ranks->resize(h->P.n_slots);
        HM_CUDA_TRY(cudaMemcpyAsync(aca_ranks->data(), h->ranks.p, sizeof(int) * h->P.n_slots, cudaMemcpyDeviceToHost,
                                    h->stream));
        HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    }
    run_phase(h, h->rec);
    HM_CUDA_TRY(cudaEventRecord(h->ev[1], h->stream));
    int f[4];
    read_flags(h, f);
    h->ms[0] = elapsed(h);
    h->assembled = true;
    h->factored = false;
    h->max_rank_C = max_rank(h);
    if (f[1] && !h->cap_hint.empty() && h->cap_retries < 3) {   // adaptive capacities: grow, retry
        regrow_caps(h);
        do_assemble(h, th);
        return;
    }
    if (f[1]) throw ApiError(HM_ERR_RANK_CAP, "assembly: a block needs more than kmax = " +
                                                  std::to_string(h->prm.kmax) + " ranks at this eps");
}

void do_cholesky(hm_handle_s* h) {
    if (!h->assembled) throw ApiError(HM_ERR_STATE, "hm_cholesky: assemble first");
    if (h->factored) throw ApiError(HM_ERR_STATE, "hm_cholesky: already factored (re-assemble first)");
    HM_CUDA_TRY(cudaMemsetAsync(h->flags.p, 0, sizeof(int) * 4, h->stream));
    HM_CUDA_TRY(cudaEventRecord(h->ev[0], h->stream));
    h->eps_run = h->eps_kc;
    run_phase(h, h->chol);
    h->eps_run = h->eps_k;
    HM_CUDA_TRY(cudaEventRecord(h->ev[1], h->stream));
    int f[4];
    read_flags(h, f);
    h->ms[1] = elapsed(h);
    h->assembled = false;   // C~ has been overwritten by L~
    if (f[0]) throw ApiError(HM_ERR_NOT_SPD, "H-Cholesky: " + std::to_string(f[0]) + " non-positive pivot(s)");
    h->factored = true;
    h->max_rank_L = max_rank(h);
    if (f[1] && !h->cap_hint.empty() && h->cap_retries < 3) {
        // adaptive capacities too small for the factor: grow them (x2, up to kmax), re-plan,
        // re-assemble at the same theta and factor again
        regrow_caps(h);
        do_assemble(h, h->theta);
        do_cholesky(h);
        return;
    }
    if (f[1]) throw ApiError(HM_ERR_RANK_CAP, "H-Cholesky: a truncation needed more than kmax ranks");
}

// Z (n x k, original order, host/device) -> out (k x 3) on host
void do_loglik(hm_handle_s* h, const double* Z, int zdev, int k, double* out_host) {
    if (!h->factored) throw ApiError(HM_ERR_STATE, "hm_loglik: call hm_cholesky first");
    const int64_t n = h->T.n;
    const int zw = h->P.zw;
    double* zt = h->pool.as<double>() + h->P.z_off;
    if ((size_t)3 * k > h->pin_out_n) {
        if (h->pin_out) HM_CUDA_TRY(cudaFreeHost(h->pin_out));
        h->pin_out = nullptr;
        HM_CUDA_TRY(cudaMallocHost(&h->pin_out, sizeof(double) * 3 * k));
        h->pin_out_n = (size_t)3 * k;
    }
    if (!zdev && (size_t)n * zw > h->pin_z_n) {
        if (h->pin_z) HM_CUDA_TRY(cudaFreeHost(h->pin_z));
        h->pin_z = nullptr;
        HM_CUDA_TRY(cudaMallocHost(&h->pin_z, sizeof(double) * n * zw));
        h->pin_z_n = (size_t)n * zw;
    }
    HM_CUDA_TRY(cudaEventRecord(h->ev[0], h->stream));
    for (int c0 = 0; c0 < k; c0 += zw) {
        const int kc = std::min(zw, k - c0);
        const double* src;
        if (zdev) {
            src = Z + (int64_t)c0 * n;
        } else {
            h->zio.alloc(sizeof(double) * n * zw);
            if (c0 > 0) HM_CUDA_TRY(cudaStreamSynchronize(h->stream));   // staging buffer reused
            std::memcpy(h->pin_z, Z + (int64_t)c0 * n, sizeof(double) * n * kc);
            HM_CUDA_TRY(cudaMemcpyAsync(h->zio.p, h->pin_z, sizeof(double) * n * kc, cudaMemcpyHostToDevice,
                                        h->stream));
            src = h->zio.as<double>();
        }
        {
            Launch L(h, KF_AUX);
            launch_gather(src, h->perm.as<int64_t>(), n, kc, zw, zt, h->stream);
        }
        {
            Launch L(h, KF_AUX);   // the solve's tile products cover only the kc active columns
            launch_set_int(h->ranks.as<int>() + h->P.z_slot, kc, h->stream);
        }
        run_phase(h, h->solve);
        {
            Launch L(h, KF_AUX);
            launch_finish(h->pool.as<double>() + h->P.logd_off, h->P.n_leaves, zt, n, kc, h->out.as<double>(),
                          h->stream);
        }
        HM_CUDA_TRY(cudaMemcpyAsync(h->pin_out + 3 * c0, h->out.p, sizeof(double) * 3 * kc, cudaMemcpyDeviceToHost,
                                    h->stream));
    }
    HM_CUDA_TRY(cudaEventRecord(h->ev[1], h->stream));
    HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    std::memcpy(out_host, h->pin_out, sizeof(double) * 3 * k);
    h->ms[2] = elapsed(h);
}

// Device bytes of a plan's task lists and ready-queue schedules (setup_device uploads).
double plan_device_bytes(const Plan& P) {
    double b = 0.0;
    for (const Phase* ph : {&P.recompress, &P.chol, &P.solve, &P.lmul})
        b += (double)ph->ins.size() * sizeof(VIns) + (double)ph->vt.size() * sizeof(VTask) +
             (double)ph->tt.size() * sizeof(TTask) + (double)ph->tp.size() * sizeof(TPiece) +
             (double)ph->terms.size() * sizeof(VTerm) + 3.0 * (double)ph->xt.size() * sizeof(XTask) +
             3.0 * (double)ph->xdeps.size() * sizeof(int32_t) + 16.0 * (double)ph->xt.size();
    return b + 8.0 * ((double)P.dgen.size() + (double)P.aca.size()) * 4.0;
}

// Adaptive capacity of a block whose C~ rank is r: 1.5 r + 8, a multiple of 4.
int32_t adaptive_cap_of(int r) { return ((r + r / 2 + 8) + 3) & ~3; }

// Plan the handle's H-Cholesky (with its capacity hints).  Device memory: if the pool (with
// the temporaries' arena planned for parallelism) and the task lists do not fit, plan again
// with an arena budget -- memory is then recycled even where that lengthens the critical
// path (plan.h build_plan).
void plan_to_fit(hm_handle_s* h) {
    const hm_params& prm = h->prm;
    const std::vector<int32_t>* hint = h->cap_hint.empty() ? nullptr : &h->cap_hint;
    build_plan(h->T, prm.kmax, h->P, prm.coop_max, INT64_MAX, hint);
    size_t fr = 0, tot = 0;
    HM_CUDA_TRY(cudaMemGetInfo(&fr, &tot));
    const double avail = 0.92 * ((double)fr + (double)h->pool.bytes) - plan_device_bytes(h->P);
    if (8.0 * (double)h->P.pool_total > avail) {
        const double budget = avail / 8.0 - (double)(h->P.pool_total - h->P.arena_size);
        if (budget < (double)(int64_t(1) << 24))
            throw ApiError(HM_ERR_OOM, "H-matrix storage does not fit in device memory (" +
                                           std::to_string(8e-9 * h->P.pool_total) + " GB needed)");
        build_plan(h->T, prm.kmax, h->P, prm.coop_max, (int64_t)budget, hint);
    }
}

// Device side of a handle whose tree and plan are built: pool, task lists, schedules.
void setup_device(hm_handle_s* h) {
    vm_set_attr();
    h->pool.alloc(sizeof(double) * (size_t)std::max<int64_t>(h->P.pool_total, 1));
    upload(h->pts, h->T.pts, h->stream);
    upload(h->perm, h->T.perm, h->stream);
    h->ranks.alloc(sizeof(int) * (h->P.n_slots + 1));
    HM_CUDA_TRY(cudaMemsetAsync(h->ranks.p, 0, sizeof(int) * (h->P.n_slots + 1), h->stream));
    h->flags.alloc(sizeof(int) * 4);
    h->ctr.alloc(sizeof(double) * CTR_N);
    {
        size_t mx = 1;
        for (const Phase* ph : {&h->P.recompress, &h->P.chol, &h->P.solve, &h->P.lmul}) mx = std::max(mx, ph->xt.size());
        h->done.alloc(sizeof(int) * mx);
        HM_CUDA_TRY(cudaMemsetAsync(h->done.p, 0, sizeof(int) * mx, h->stream));
        h->counter.alloc(sizeof(int) * 4);
        h->rq_cnt.alloc(sizeof(int) * mx);
        h->rq_slot.alloc(sizeof(int) * mx);
        h->rq_ctl.alloc(sizeof(int) * (2 * RQ_NQ + 2));
        int nb = 1;
        for (const Phase* ph : {&h->P.recompress, &h->P.chol, &h->P.solve, &h->P.lmul}) nb = std::max(nb, ph->n_bars);
        h->bars.alloc(sizeof(int) * nb);
        exec_grid();
        exec_grid_rq();
    }
    HM_CUDA_TRY(cudaMemsetAsync(h->ctr.p, 0, sizeof(double) * CTR_N, h->stream));
    h->out.alloc(sizeof(double) * 3 * h->P.zw);
    upload(h->dgen, h->P.dgen, h->stream);
    upload(h->aca, h->P.aca, h->stream);
    upload_phase(h->rec, h->P.recompress, h->stream);
    upload_phase(h->chol, h->P.chol, h->stream);
    upload_phase(h->solve, h->P.solve, h->stream);
    upload_phase(h->lmul, h->P.lmul, h->stream);
}


// ---- co-scheduled evaluations (hm_loglik_batch, hm_loglik_multi) ----------
int max_group(const hm_handle_s* h) {
    return std::max(std::max(h->rec.max_nsub, h->chol.max_nsub), std::max(h->solve.max_nsub, h->lmul.max_nsub));
}
// CTAs an executor needs so that groups partially claimed by waiting CTAs never
// exhaust it (exec.cu: grid > RQ_NCOOP * (largest group - 1))
int ctas_needed(const hm_handle_s* h) { return RQ_NCOOP * (max_group(h) - 1) + 1; }

hm_handle_s* clone_handle(const hm_handle_s* p) {
    std::unique_ptr<hm_handle_s> h(new hm_handle_s());
    h->device = p->device;
    h->prm = p->prm;
    h->poison = p->poison;
    h->abs_eps = p->abs_eps;
    h->exec_mode = p->exec_mode;
    HM_CUDA_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
    HM_CUDA_TRY(cudaEventCreate(&h->ev[0]));
    HM_CUDA_TRY(cudaEventCreate(&h->ev[1]));
    h->T = p->T;
    h->P = p->P;
    h->cap_hint = p->cap_hint;
    setup_device(h.get());
    HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    return h.release();
}

struct Job {
    hm_handle_s* bound;   // executor that must run it (hm_loglik_multi) or nullptr (any)
    hm_theta th;
    const double* Z;
    double* out;          // k x 3
};

// One host thread per executor handle, the persistent executors splitting the SMs
// (each capped at total / S CTAs for the call).  A job's failure stores
// (-inf, nan, nan) for its columns; the first error is returned.
int run_jobs(std::vector<hm_handle_s*>& ex, std::vector<Job>& jobs, int zdev, int k) {
    const int S = (int)ex.size();
    const int total = exec_grid_rq();
    std::vector<int> oldcap(S);
    for (int i = 0; i < S; ++i) {
        oldcap[i] = ex[i]->exec_grid_cap;
        ex[i]->exec_grid_cap = S > 1 ? total / S + (i < total % S ? 1 : 0) : oldcap[i];
        if (S > 1 && ex[i]->exec_grid_cap < ctas_needed(ex[i])) {
            for (int j = 0; j <= i; ++j) ex[j]->exec_grid_cap = oldcap[j];
            throw ApiError(HM_ERR_ARG, "co-scheduling " + std::to_string(S) + " evaluations leaves " +
                                           std::to_string(total / S) + " CTAs per executor, the plan's cooperative "
                                           "truncations need " + std::to_string(ctas_needed(ex[i])) +
                                           " (build with a smaller coop_max)");
        }
    }
    std::atomic<int> next{0};
    std::mutex mu;
    int first = HM_OK;
    std::string msg;
    auto fail = [&](int rc, const std::string& m) {
        std::lock_guard<std::mutex> lk(mu);
        if (first == HM_OK) {
            first = rc;
            msg = m;
        }
    };
    auto run_one = [&](hm_handle_s* h, const Job& j) {
        try {
            do_assemble(h, j.th);
            do_cholesky(h);
            do_loglik(h, j.Z, zdev, k, j.out);
        } catch (...) {
            const int rc = translate_exception();
            fail(rc, hm_last_error());
            for (int c = 0; c < k; ++c) {
                j.out[3 * c] = -std::numeric_limits<double>::infinity();
                j.out[3 * c + 1] = j.out[3 * c + 2] = std::numeric_limits<double>::quiet_NaN();
            }
        }
    };
    auto worker = [&](int i) {
        hm_handle_s* h = ex[i];
        if (cudaSetDevice(h->device) != cudaSuccess) {
            fail(HM_ERR_CUDA, "cudaSetDevice failed in a co-scheduling thread");
            return;
        }
        if (jobs.empty()) return;
        if (jobs[0].bound) {   // bound jobs: executor i runs the jobs bound to it
            for (const Job& j : jobs)
                if (j.bound == h) run_one(h, j);
            return;
        }
        for (int q = next++; q < (int)jobs.size(); q = next++) run_one(h, jobs[q]);
    };
    std::vector<std::thread> th;
    for (int i = 1; i < S; ++i) th.emplace_back(worker, i);
    worker(0);
    for (auto& t : th) t.join();
    for (int i = 0; i < S; ++i) {
        ex[i]->exec_grid_cap = oldcap[i];
        ex[i]->assembled = ex[i]->factored = false;   // state after a batch: assemble again
    }
    if (first != HM_OK) set_error(first, msg);
    return first;
}

}  // namespace

extern "C" {

int hm_build(const double* locs, int32_t locs_on_device, int64_t n, hm_theta theta, hm_params params, int32_t device,
             void* stream, hm_handle* out) {
    hm_handle_s* h = nullptr;
    bool probing = false;   // adaptive capacities: a rank cap in the probe is fatal (no factor plan yet)
    try {
        if (!locs || !out) throw ApiError(HM_ERR_ARG, "null pointer");
        if (n < 1) throw ApiError(HM_ERR_ARG, "n >= 1 required");
        if (!(params.eps > 0.0 && params.eps < 1.0)) throw ApiError(HM_ERR_ARG, "0 < eps < 1 required");
        if (params.eps_chol == 0.0) params.eps_chol = params.eps;
        if (!(params.eps_chol > 0.0 && params.eps_chol < 1.0)) throw ApiError(HM_ERR_ARG, "0 < eps_chol < 1 required");
        if (params.leaf < 1 || params.leaf > 128) throw ApiError(HM_ERR_ARG, "1 <= leaf <= 128 required");
        if (!(params.eta > 0.0)) throw ApiError(HM_ERR_ARG, "eta > 0 required");
        if (params.kmax <= 0) params.kmax = 160;
        if (params.coop_max <= 0) params.coop_max = TR_COOP_DEFAULT;
        if (params.coop_max > TR_COOP_MAX) throw ApiError(HM_ERR_ARG, "coop_max <= 32 required");
        if (params.kmax > HM_KMAX_LIMIT) throw ApiError(HM_ERR_ARG, "kmax <= 240 required");
        if (params.exec_ctas < 0) throw ApiError(HM_ERR_ARG, "exec_ctas >= 0 required");
        if (params.adaptive_cap < 0 || params.adaptive_cap > 1) throw ApiError(HM_ERR_ARG, "adaptive_cap must be 0 or 1");
        check_theta(theta);
        DeviceGuard dg(device);
        h = new hm_handle_s();
        h->device = device;
        h->prm = params;
        if (const char* pz = std::getenv("HM_POISON_RING")) h->poison = pz[0] == '1';
        h->abs_eps = params.rel_eps == 0;
        h->exec_grid_cap = params.exec_ctas;
        if (stream) {
            h->stream = (cudaStream_t)stream;
        } else {
            HM_CUDA_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
            h->own_stream = true;
        }
        HM_CUDA_TRY(cudaEventCreate(&h->ev[0]));
        HM_CUDA_TRY(cudaEventCreate(&h->ev[1]));
        std::vector<double> hl;
        const double* hp = locs;
        if (locs_on_device) {
            hl.resize(2 * n);
            HM_CUDA_TRY(cudaMemcpy(hl.data(), locs, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
            hp = hl.data();
        }
        build_tree(hp, n, params.leaf, params.eta, h->T);
        if (params.adaptive_cap) {
            probing = true;
            // rank probe: assemble C~ at capacity kmax with an assembly-only plan, then size
            // every low-rank block from its C~ rank (the factor's ranks run somewhat higher)
            build_plan(h->T, params.kmax, h->P, params.coop_max, INT64_MAX, nullptr, true);
            setup_device(h);
            std::vector<int> aca_r;
            do_assemble(h, theta, &aca_r);
            h->cap_hint.assign(h->P.bs.size(), 0);
            // HM_ADAPTIVE_SCALE (tests): scale the capacities down to exercise the regrowth path
            const double sc = std::getenv("HM_ADAPTIVE_SCALE") ? std::atof(std::getenv("HM_ADAPTIVE_SCALE")) : 1.0;
            for (size_t b = 0; b < h->P.bs.size(); ++b)
                if (h->P.bs[b].kind == ST_LR) {
                    // room for the factor's rank (1.5 r + 8) and for ACA's iterations before recompression
                    const int rs = h->P.bs[b].rslot;
                    const int c = std::max(adaptive_cap_of(h->h_ranks[rs]), (aca_r[rs] + 2 + 3) & ~3);
                    h->cap_hint[b] = std::max(1, (int)(sc * c));
                }
            h->pool.release();
            probing = false;
        }
        plan_to_fit(h);
        setup_device(h);
        do_assemble(h, theta);
        *out = h;
        return HM_OK;
    } catch (...) {
        int rc = translate_exception();
        if (rc == HM_ERR_RANK_CAP && h && !probing) {   // handle is usable; report the cap
            *out = h;
            return rc;
        }
        delete h;
        return rc;
    }
}

int hm_free(hm_handle h) {
    delete h;
    return HM_OK;
}

int hm_assemble(hm_handle h, hm_theta theta) {
    try {
        if (!h) throw ApiError(HM_ERR_ARG, "null handle");
        DeviceGuard dg(h->device);
        do_assemble(h, theta);
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_cholesky(hm_handle h) {
    try {
        if (!h) throw ApiError(HM_ERR_ARG, "null handle");
        DeviceGuard dg(h->device);
        do_cholesky(h);
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_loglik(hm_handle h, const double* Z, int32_t z_on_device, int32_t k, double* out_host) {
    try {
        if (!h || !Z || !out_host) throw ApiError(HM_ERR_ARG, "null pointer");
        if (k < 1) throw ApiError(HM_ERR_ARG, "k >= 1 required");
        DeviceGuard dg(h->device);
        do_loglik(h, Z, z_on_device, k, out_host);
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_loglik_batch(hm_handle h, const hm_theta* thetas, int32_t n_theta, const double* Z, int32_t z_on_device,
                    int32_t k, double* out_host) {
    try {
        if (!h || !thetas || !Z || !out_host) throw ApiError(HM_ERR_ARG, "null pointer");
        if (k < 1 || n_theta < 0) throw ApiError(HM_ERR_ARG, "k >= 1, n_theta >= 0 required");
        DeviceGuard dg(h->device);
        for (int i = 0; i < n_theta; ++i) check_theta(thetas[i]);
        // S co-scheduled executors: the handle + S - 1 siblings on the same tree and plan
        const int total = exec_grid_rq();
        int S = h->batch_streams > 0 ? h->batch_streams : 4;
        S = std::max(1, std::min(S, total / ctas_needed(h)));
        S = std::min(S, std::max(1, n_theta));
        try {
            while ((int)h->subs.size() < S - 1) h->subs.emplace_back(clone_handle(h));
        } catch (const ApiError& e) {   // out of device memory: co-schedule what exists
            if (e.code != HM_ERR_OOM) throw;
            S = 1 + (int)h->subs.size();
        }
        std::vector<hm_handle_s*> ex{h};
        for (int i = 0; i < S - 1; ++i) ex.push_back(h->subs[i].get());
        std::vector<Job> jobs;
        for (int i = 0; i < n_theta; ++i) jobs.push_back(Job{nullptr, thetas[i], Z, out_host + (int64_t)3 * k * i});
        return run_jobs(ex, jobs, z_on_device, k);
    } catch (...) {
        return translate_exception();
    }
}

int hm_loglik_multi(int32_t nh, const hm_handle* hs, const hm_theta* thetas, const double* const* Zs,
                    int32_t z_on_device, int32_t k, double* out_host) {
    try {
        if (nh < 1 || !hs || !thetas || !Zs || !out_host) throw ApiError(HM_ERR_ARG, "null pointer or nh < 1");
        if (k < 1) throw ApiError(HM_ERR_ARG, "k >= 1 required");
        std::vector<hm_handle_s*> ex;
        std::vector<Job> jobs;
        for (int i = 0; i < nh; ++i) {
            if (!hs[i] || !Zs[i]) throw ApiError(HM_ERR_ARG, "null handle or data pointer");
            if (hs[i]->device != hs[0]->device) throw ApiError(HM_ERR_ARG, "all handles must be on one device");
            for (int j = 0; j < i; ++j)
                if (hs[j] == hs[i]) throw ApiError(HM_ERR_ARG, "a handle appears twice");
            check_theta(thetas[i]);
            ex.push_back(hs[i]);
            jobs.push_back(Job{hs[i], thetas[i], Zs[i], out_host + (int64_t)3 * k * i});
        }
        DeviceGuard dg(hs[0]->device);
        return run_jobs(ex, jobs, z_on_device, k);
    } catch (...) {
        return translate_exception();
    }
}

int hm_set_batch_streams(hm_handle h, int32_t streams) {
    if (!h) return set_error(HM_ERR_ARG, "null handle");
    if (streams < 0 || streams > 16) return set_error(HM_ERR_ARG, "streams must be in [0, 16]");
    h->batch_streams = streams;
    if (streams > 0)
        while ((int)h->subs.size() > streams - 1) h->subs.pop_back();   // release surplus siblings
    return HM_OK;
}

int hm_sample(hm_handle h, const double* xi, int32_t xi_on_device, int32_t k, double* Z, int32_t z_on_device) {
    try {
        if (!h || !xi || !Z) throw ApiError(HM_ERR_ARG, "null pointer");
        if (k < 1) throw ApiError(HM_ERR_ARG, "k >= 1 required");
        if (!h->factored) throw ApiError(HM_ERR_STATE, "hm_sample: call hm_cholesky first");
        DeviceGuard dg(h->device);
        const int64_t n = h->T.n;
        const int zw = h->P.zw;
        double* zt = h->pool.as<double>() + h->P.z_off;
        h->zio.alloc(sizeof(double) * n * zw);
        for (int c0 = 0; c0 < k; c0 += zw) {
            const int kc = std::min(zw, k - c0);
            const double* src = xi + (int64_t)c0 * n;
            if (!xi_on_device) {
                HM_CUDA_TRY(cudaMemcpyAsync(h->zio.p, src, sizeof(double) * n * kc, cudaMemcpyHostToDevice, h->stream));
                src = h->zio.as<double>();
            }
            launch_gather(src, h->perm.as<int64_t>(), n, kc, zw, zt, h->stream);
            launch_set_int(h->ranks.as<int>() + h->P.z_slot, kc, h->stream);
            run_phase(h, h->lmul);
            if (z_on_device) {
                launch_scatter(zt, h->perm.as<int64_t>(), n, kc, Z + (int64_t)c0 * n, h->stream);
            } else {
                launch_scatter(zt, h->perm.as<int64_t>(), n, kc, h->zio.as<double>(), h->stream);
                HM_CUDA_TRY(cudaMemcpyAsync(Z + (int64_t)c0 * n, h->zio.p, sizeof(double) * n * kc,
                                            cudaMemcpyDeviceToHost, h->stream));
            }
        }
        HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}


int hm_stats(hm_handle h, double st[12]) {
    try {
        if (!h || !st) throw ApiError(HM_ERR_ARG, "null pointer");
        const Plan& P = h->P;
        int64_t nd = 0, nl = 0;
        double bytesC = 0, bytesL = 0;
        DeviceGuard dg(h->device);
        max_rank(h);
        for (size_t b = 0; b < P.bs.size(); ++b) {
            const BStore& s = P.bs[b];
            if (s.kind == ST_DENSE) {
                ++nd;
                bytesC += 8.0 * s.m * s.p;
            } else if (s.kind == ST_LR) {
                ++nl;
                bytesC += 8.0 * (s.m + s.p) * h->h_ranks[s.rslot];
            }
        }
        bytesL = bytesC;   // storage of whatever the handle currently holds (C~ or L~)
        const double n = (double)h->T.n;
        st[0] = n;
        st[1] = (double)nd;
        st[2] = (double)nl;
        st[3] = h->max_rank_C;
        st[4] = h->max_rank_L;
        st[5] = bytesC;
        st[6] = bytesL;
        st[7] = 1.0 - bytesC / (8.0 * n * n);
        st[8] = (double)(P.chol.vt.size() + P.chol.tt.size());
        st[9] = P.chol.nwaves;
        st[10] = (double)P.chol.n_launches();
        // widest truncation of the Cholesky at the current ranks (sum of actual piece widths)
        int kmaxw = 0;
        for (const TTask& t : P.chol.tt) {
            int K = 0;
            for (int p = 0; p < t.piece_count; ++p) {
                const Dim& d = P.chol.tp[t.piece_begin + p].w;
                if (d.slot < 0) K += d.stat;
                else K += std::max(0, std::min(d.stat, h->h_ranks[d.slot] - d.off));
            }
            kmaxw = std::max(kmaxw, K);
        }
        st[11] = kmaxw;
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

static void profile_one(hm_handle_s* h, bool on) {
    HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    h->profiling = on;
    h->evlog.clear();
    // create the event pool up front: creating events while other streams run kernels
    // serialises co-scheduled handles (measured: 2 streams 2.69 -> 1.46 evals/s)
    while (h->profiling && h->evpool.size() < 4096) {
        cudaEvent_t e;
        HM_CUDA_TRY(cudaEventCreate(&e));
        h->evpool.push_back(e);
    }
    for (auto& x : h->launches) x = 0;
    HM_CUDA_TRY(cudaMemsetAsync(h->ctr.p, 0, sizeof(double) * CTR_N, h->stream));
    HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
}

int hm_profile(hm_handle h, int32_t enable) {
    try {
        if (!h) throw ApiError(HM_ERR_ARG, "null handle");
        DeviceGuard dg(h->device);
        profile_one(h, enable != 0);
        for (auto& sb : h->subs) profile_one(sb.get(), enable != 0);   // hm_loglik_batch siblings
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_checksum(hm_handle h, double out[4]) {
    try {
        if (!h || !out) throw ApiError(HM_ERR_ARG, "null pointer");
        DeviceGuard dg(h->device);
        HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
        const Plan& P = h->P;
        std::vector<double> pool((size_t)P.pool_blocks);
        HM_CUDA_TRY(cudaMemcpy(pool.data(), h->pool.p, sizeof(double) * pool.size(), cudaMemcpyDeviceToHost));
        max_rank(h);
        double sd = 0, sl = 0, sr = 0, sw = 0;
        for (size_t b = 0; b < P.bs.size(); ++b) {
            const BStore& st = P.bs[b];
            if (st.kind == ST_DENSE) {
                for (int64_t i = 0; i < (int64_t)st.m * st.p; ++i) {
                    sd += std::fabs(pool[st.d_off + i]);
                    sw += pool[st.d_off + i] * (double)((i % 97) + 1);
                }
            } else if (st.kind == ST_LR) {
                const int r = h->h_ranks[st.rslot];
                sr += r;
                for (int64_t i = 0; i < (int64_t)st.m * r; ++i) sl += std::fabs(pool[st.u_off + i]);
                for (int64_t i = 0; i < (int64_t)st.p * r; ++i) sl += std::fabs(pool[st.v_off + i]);
            }
        }
        out[0] = sd; out[1] = sw; out[2] = sl; out[3] = sr;
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_to_dense(hm_handle h, double* out) {
    try {
        if (!h || !out) throw ApiError(HM_ERR_ARG, "null pointer");
        const int64_t n = h->T.n;
        if (n > HM_DENSE_NMAX) throw ApiError(HM_ERR_TOO_LARGE, "hm_to_dense: n above HM_DENSE_NMAX");
        if (!h->assembled && !h->factored) throw ApiError(HM_ERR_STATE, "hm_to_dense: nothing assembled");
        DeviceGuard dg(h->device);
        HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
        const Plan& P = h->P;
        std::vector<double> pool((size_t)P.pool_blocks);
        HM_CUDA_TRY(cudaMemcpy(pool.data(), h->pool.p, sizeof(double) * pool.size(), cudaMemcpyDeviceToHost));
        max_rank(h);
        const bool lower = h->factored;   // L~: lower triangular; C~: symmetric
        std::vector<double> M((size_t)(n * n), 0.0);   // tree order, column-major
        auto put = [&](int64_t i, int64_t j, double v) {
            if (i == j || i > j) M[(size_t)(i + j * n)] = v;
            if (!lower && i != j) M[(size_t)(j + i * n)] = v;
        };
        for (const DenseGenTask& d : P.dgen)
            for (int64_t j = 0; j < d.q; ++j)
                for (int64_t i = 0; i < d.m; ++i) {
                    const int64_t gi = d.r0 + i, gj = d.c0 + j;
                    if (gi < gj) continue;   // diagonal blocks: upper part is mirrored / zero
                    put(gi, gj, pool[(size_t)(d.off + i + j * d.m)]);
                }
        for (const AcaTask& a : P.aca) {
            const int r = h->h_ranks[a.rslot];
            for (int64_t j = 0; j < a.q; ++j)
                for (int64_t i = 0; i < a.m; ++i) {
                    double v = 0.0;
                    for (int k = 0; k < r; ++k)
                        v += pool[(size_t)(a.u_off + i + (int64_t)k * a.m)] * pool[(size_t)(a.v_off + j + (int64_t)k * a.q)];
                    put(a.r0 + i, a.c0 + j, v);
                }
        }
        const int64_t* pm = h->T.perm.data();
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) out[pm[i] + pm[j] * n] = M[(size_t)(i + j * n)];
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_trace(hm_handle h, int32_t enable, const char* path) {
    try {
        if (!h) throw ApiError(HM_ERR_ARG, "null handle");
        DeviceGuard dg(h->device);
        HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
        if (path && h->trace_n > 0) {
            std::vector<unsigned long long> buf(68 * (size_t)h->trace_n);
            HM_CUDA_TRY(cudaMemcpy(buf.data(), h->trace.p, buf.size() * 8, cudaMemcpyDeviceToHost));
            FILE* f = std::fopen(path, "wb");
            if (!f) throw ApiError(HM_ERR_ARG, std::string("cannot open ") + path);
            std::fwrite(buf.data(), 8, buf.size(), f);
            std::fclose(f);
        }
        if (enable) {
            size_t mx = 1;
            for (const Phase* ph : {&h->P.recompress, &h->P.chol, &h->P.solve, &h->P.lmul}) mx = std::max(mx, ph->xt.size());
            h->trace.alloc(8 * 68 * mx);   // 4 per task + 64 truncation stage stamps per task
        }
        h->tracing = enable != 0;
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_set_exec_mode(hm_handle h, int32_t mode) {
    if (!h) return set_error(HM_ERR_ARG, "null handle");
    if (mode < 0 || mode > 2)
        return set_error(HM_ERR_ARG, "mode must be 0 (waves), 1 (persistent, topological claim) or 2 (persistent, ready queues)");
    h->exec_mode = mode;
    return HM_OK;
}

int hm_set_exec_grid(hm_handle h, int32_t ctas) {
    if (!h) return set_error(HM_ERR_ARG, "null handle");
    if (ctas < 0) return set_error(HM_ERR_ARG, "ctas must be >= 0");
    h->exec_grid_cap = ctas;
    return HM_OK;
}

static void kernel_stats_one(hm_handle_s* h, double out[24]) {
    HM_CUDA_TRY(cudaStreamSynchronize(h->stream));
    double ms[KF_N] = {0, 0, 0, 0, 0, 0};
    for (auto& e : h->evlog) {
        float t = 0;
        HM_CUDA_TRY(cudaEventElapsedTime(&t, h->evpool[e.second], h->evpool[e.second + 1]));
        ms[e.first] += t;
    }
    double c[CTR_N];
    HM_CUDA_TRY(cudaMemcpy(c, h->ctr.p, sizeof(double) * CTR_N, cudaMemcpyDeviceToHost));
    const int cmap[KF_N] = {CTR_DGEN, CTR_ACA, CTR_TRUNC, CTR_VM, -1, -1};
    for (int f = 0; f < KF_N; ++f) {
        out[4 * f + 0] += (double)h->launches[f];
        out[4 * f + 1] += ms[f];
        out[4 * f + 2] += cmap[f] >= 0 ? c[cmap[f]] : 0.0;
        out[4 * f + 3] += cmap[f] >= 0 ? c[cmap[f] + 1] : 0.0;
    }
    // the persistent executor runs the truncation and tile-VM tasks: its work is theirs
    out[4 * KF_EXEC + 2] += c[CTR_TRUNC] + c[CTR_VM];
    out[4 * KF_EXEC + 3] += c[CTR_TRUNC + 1] + c[CTR_VM + 1];
}

int hm_kernel_stats(hm_handle h, double out[24]) {
    try {
        if (!h || !out) throw ApiError(HM_ERR_ARG, "null pointer");
        DeviceGuard dg(h->device);
        for (int i = 0; i < 24; ++i) out[i] = 0.0;
        kernel_stats_one(h, out);
        for (auto& sb : h->subs) kernel_stats_one(sb.get(), out);   // hm_loglik_batch siblings
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_timings(hm_handle h, double ms[3]) {
    if (!h || !ms) return set_error(HM_ERR_ARG, "null pointer");
    for (int i = 0; i < 3; ++i) ms[i] = h->ms[i];
    return HM_OK;
}

}  // extern "C"

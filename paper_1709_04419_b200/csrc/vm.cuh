// Tile VM: one CTA executes a short program (hm_tasks.h VmOp) on NTILE 64 x 64
// fp64 shared-memory tiles -- leaf-level POTRF / TRSM / TRMM and the products of
// the H-Cholesky, solves and sampler (sec. 3.1, l.259-283).
#pragma once
#include <cuda_runtime.h>

#include "dev_util.cuh"
#include "hm_kernels.h"
#include "hm_tasks.h"
#include "gemm.cuh"
#include "tile.cuh"

namespace hm {

// VM_MGEMM: T0 (64 x 64 smem tile) += sum_t alpha_t op(A_t) op(B_t).  The (term, 16-wide
// K chunk) sequence of all terms is streamed global -> shared memory through a
// VM_NS-stage cp.async pipeline (zero-filled outside each operand's dims) into
// the staging area behind the NTILE tiles (VM_SMEM), and accumulated in registers by the FP64 tensor
// cores (warp tile 16 x 32, 4 x 2 warps); T0 is updated once at the end.
struct TermRt {
    const double* a;
    const double* b;
    int32_t lda, ldb, M, N, K, ch0;   // op(A) M x K, op(B) K x N; first chunk index
    int32_t ta, tb;
    int32_t va, vb;                   // operand staged with 16-byte copies (aligned, even ld)
    double alpha;
};

// One operand's K chunk (rows [0, R) x k in [k0, k0 + GM_BK) of op(X), K columns in all)
// into a stage: kc = contiguous along k (X^T of a column-major A, or B), staged [row][k]
// with ld 20, else [k][row] with ld 68; vec = 16-byte element pairs along the contiguous
// dimension, else 8-byte copies; zero-filled outside the operand.
constexpr int VM_NS = 4;                         // pipeline stages
constexpr int VM_STAGE = 64 * 20;                // doubles per stage (>= GM_BK * 68)
static_assert(GM_BK * 68 <= VM_STAGE, "stage holds either layout");
constexpr int VM_SMEM = (NTILE * TSZ + 2 * VM_NS * VM_STAGE) * 8;   // bytes: tiles + A / B stages
__device__ __forceinline__ void vm_stage(double* st, const double* p, int64_t ld, bool kc, bool vec, int R, int K,
                                         int k0) {
    if (vec) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {                    // 512 pairs = 64 x 16 / 2
            const int pr = threadIdx.x + e * 256;
            int r, k, so, n;
            if (kc) {
                k = 2 * (pr & 7); r = pr >> 3; so = r * 20 + k;
                const int left = K - k0 - k;
                n = (r < R) ? (left >= 2 ? 2 : (left > 0 ? left : 0)) : 0;
            } else {
                r = 2 * (pr & 31); k = pr >> 5; so = k * 68 + r;
                n = (k0 + k < K) ? (r + 1 < R ? 2 : (r < R ? 1 : 0)) : 0;
            }
            const double* src = kc ? p + (k0 + k) + (int64_t)r * ld : p + r + (int64_t)(k0 + k) * ld;
            cp_async16(st + so, n ? src : p, 8 * n);
        }
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int idx = threadIdx.x + e * 256;       // 1024 = 64 x 16
            int r, k, so;
            if (kc) { k = idx & 15; r = idx >> 4; so = r * 20 + k; }
            else { r = idx & 63; k = idx >> 6; so = k * 68 + r; }
            const bool ok = r < R && k0 + k < K;
            cp_async8(st + so, ok ? (kc ? p + (k0 + k) + (int64_t)r * ld : p + r + (int64_t)(k0 + k) * ld) : p, ok);
        }
    }
}

// dst == nullptr: T0 += result (smem tile); else dst[r + c ldd] = beta dst + result for
// r < drows, c < dcols (VM_MGEMM_ST: accumulators straight to global memory)
__device__ __forceinline__ void vm_mgemm(double* T0, const VTerm* __restrict__ terms, int nt, const double* pool,
                                         const int* ranks, double* stageA, double* stageB, double& c_fl, double& c_by,
                                         double* dst = nullptr, int64_t ldd = 0, int drows = 0, int dcols = 0,
                                         double beta = 0.0, unsigned long long* stt = nullptr) {
    // staged chunks: an operand contiguous along the tile dimension (A, B^T) as [k][row]
    // with ld 68, one contiguous along k (A^T, B) as [row][k] with ld 20 -- both keep rows
    // 16-byte aligned for 16-byte copies of element pairs and make the fragment loads
    // conflict-free (bank offsets 8t + 2g resp. 8g + 2t per half-warp)
    constexpr int SA = VM_STAGE, SB = VM_STAGE;
    __shared__ TermRt tr[VM_MAX_TERMS];
    __shared__ int s_nch;
    if (threadIdx.x < nt) {
        const VTerm v = terms[threadIdx.x];
        const int ar = dim_eval(v.a_rows, ranks), ac = dim_eval(v.a_cols, ranks);
        const int br = dim_eval(v.b_rows, ranks), bc = dim_eval(v.b_cols, ranks);
        TermRt r;
        r.a = pool + v.a_off;
        r.b = pool + v.b_off;
        r.lda = v.a_ld;
        r.ldb = v.b_ld;
        r.ta = v.ta;
        r.tb = v.tb;
        r.M = v.ta ? ac : ar;
        r.N = v.tb ? br : bc;
        const int ka = v.ta ? ar : ac, kb = v.tb ? bc : br;
        r.K = ka < kb ? ka : kb;
        r.alpha = v.alpha;
        r.va = ((reinterpret_cast<uintptr_t>(r.a) & 15) == 0) && ((v.a_ld & 1) == 0);
        r.vb = ((reinterpret_cast<uintptr_t>(r.b) & 15) == 0) && ((v.b_ld & 1) == 0);
        tr[threadIdx.x] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = 0;
        for (int t = 0; t < nt; ++t) {
            tr[t].ch0 = c;
            c += (tr[t].K + GM_BK - 1) / GM_BK;
            c_fl += 2.0 * tr[t].M * tr[t].N * tr[t].K;
            c_by += 8.0 * ((double)tr[t].M + tr[t].N) * tr[t].K;
        }
        s_nch = c;
        if (stt) stt[2] = gtimer();
    }
    __syncthreads();
    const int nch = s_nch;
    double* As = stageA;                                 // VM_NS stages each (exec.cu: behind the tiles)
    double* Bs = stageB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm = (warp >> 1) * 16, wn = (warp & 1) * 32;
    double acc[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    int it = 0;                                          // issue cursor: term / chunk within it
    int ik = 0;
    auto issue = [&](int s) {
        while (it < nt && ik >= (tr[it].K + GM_BK - 1) / GM_BK) { ++it; ik = 0; }
        const TermRt r = tr[it];
        const int k0 = ik * GM_BK;
        double* as = As + (s % VM_NS) * SA;
        double* bs = Bs + (s % VM_NS) * SB;
        vm_stage(as, r.a, r.lda, r.ta != 0, r.va != 0, r.M, r.K, k0);
        vm_stage(bs, r.b, r.ldb, r.tb == 0, r.vb != 0, r.N, r.K, k0);
        ++ik;
    };
    int ct = 0, ck = 0;                                  // compute cursor
    auto compute = [&](int s) {
        while (ct < nt && ck >= (tr[ct].K + GM_BK - 1) / GM_BK) { ++ct; ck = 0; }
        const double al = tr[ct].alpha;
        const bool kcA = tr[ct].ta != 0, kcB = tr[ct].tb == 0;
        // fragments outside this term's op(A) rows / op(B) columns get zeros from it: skip
        // their DMMAs (warp-uniform; low-rank factors are often much narrower than 64)
        const int am = tr[ct].M - wm, bn = tr[ct].N - wn, kr = tr[ct].K - ck * GM_BK;
        ++ck;
        if (am <= 0 || bn <= 0) return;
        const double* as = As + (s % VM_NS) * SA;
        const double* bs = Bs + (s % VM_NS) * SB;
#pragma unroll
        for (int kk = 0; kk < GM_BK; kk += 4) {
            if (kk >= kr) break;
            double af[2], bf[4];
#pragma unroll
            for (int a = 0; a < 2; ++a) af[a] = al * as[kcA ? (wm + a * 8 + g) * 20 + kk + t4 : (kk + t4) * 68 + wm + a * 8 + g];
#pragma unroll
            for (int b = 0; b < 4; ++b) bf[b] = bs[kcB ? (wn + b * 8 + g) * 20 + kk + t4 : (kk + t4) * 68 + wn + b * 8 + g];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (a * 8 < am && b * 8 < bn) dmma_884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
    };
    if (nch <= VM_NS) {
        // short sums (the latency-bound tasks on the Cholesky's critical path): every chunk
        // in flight at once, a single wait
        for (int s = 0; s < nch; ++s) issue(s);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        for (int s = 0; s < nch; ++s) compute(s);
    } else {
#pragma unroll
        for (int s = 0; s < VM_NS - 1; ++s) {
            issue(s);
            cp_async_commit();
        }
        for (int s = 0; s < nch; ++s) {
            cp_async_wait<VM_NS - 2>();
            __syncthreads();
            if (s + VM_NS - 1 < nch) issue(s + VM_NS - 1);
            cp_async_commit();
            compute(s);
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    if (stt && threadIdx.x == 0) stt[3] = gtimer();
    if (dst) {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int r = wm + a * 8 + g, c = wn + b * 8 + 2 * t4;
                if (r < drows) {
                    if (c < dcols) {
                        double* p = dst + r + (int64_t)c * ldd;
                        *p = (beta != 0.0 ? beta * __ldcg(p) : 0.0) + acc[a][b][0];
                    }
                    if (c + 1 < dcols) {
                        double* p = dst + r + (int64_t)(c + 1) * ldd;
                        *p = (beta != 0.0 ? beta * __ldcg(p) : 0.0) + acc[a][b][1];
                    }
                }
            }
        if (threadIdx.x == 0) c_by += 8.0 * drows * dcols * (beta != 0.0 ? 2.0 : 1.0);
        __syncthreads();
        if (stt && threadIdx.x == 0) stt[4] = gtimer();
        return;
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int r = wm + a * 8 + g, c = wn + b * 8 + 2 * t4;
            T0[c * TLD + r] += acc[a][b][0];
            T0[(c + 1) * TLD + r] += acc[a][b][1];
        }
    __syncthreads();
}

// Execute one tile-VM program with the CTA (TTHREADS threads); sm = NTILE tiles.
__device__ __forceinline__ void vm_run(const VTask task, const VIns* __restrict__ ins, const VTerm* __restrict__ terms,
                                       double* pool, const int* ranks, int* flags, double* ctr, double* sm,
                                       unsigned long long* stt = nullptr) {
    __shared__ int trows[NTILE], tcols[NTILE];
    if (stt && threadIdx.x == 0) stt[0] = gtimer();
    __shared__ double s_log;
    double c_fl = 0.0, c_by = 0.0;   // algorithmic flops / bytes of this program (thread 0)
    for (int pc = 0; pc < task.ins_count; ++pc) {
        const VIns I = ins[task.ins_begin + pc];
        if (stt && pc == 0 && threadIdx.x == 0) stt[1] = gtimer();
        double* T0 = sm + (int)I.t0 * TSZ;
        switch (I.op) {
            case VM_LD: {
                const int r = dim_eval(I.rows, ranks), c = dim_eval(I.cols, ranks);
                tile_load(T0, pool + I.goff, I.ld, r, c);
                if (threadIdx.x == 0) { trows[I.t0] = r; tcols[I.t0] = c; c_by += 8.0 * r * c; }
                __syncthreads();
            } break;
            case VM_ST: {
                const int r = dim_eval(I.rows, ranks), c = dim_eval(I.cols, ranks);
                tile_store(T0, pool + I.goff, I.ld, min(r, trows[I.t0]), min(c, tcols[I.t0]));
                if (threadIdx.x == 0) c_by += 8.0 * min(r, trows[I.t0]) * min(c, tcols[I.t0]);
                __syncthreads();
            } break;
            case VM_MGEMM: {
                vm_mgemm(T0, terms + I.goff, I.ld, pool, ranks, sm + NTILE * TSZ, sm + NTILE * TSZ + VM_NS * VM_STAGE,
                         c_fl, c_by);
            } break;
            case VM_MGEMM_ST: {
                const int r = dim_eval(I.rows, ranks), c = dim_eval(I.cols, ranks);
                vm_mgemm(T0, terms + I.pad2, I.t1, pool, ranks, sm + NTILE * TSZ, sm + NTILE * TSZ + VM_NS * VM_STAGE,
                         c_fl, c_by, pool + I.goff,
                         I.ld, r, c, I.beta, task.ins_count == 1 ? stt : nullptr);
            } break;
            case VM_ADD: {
                if (threadIdx.x == 0) c_fl += (double)trows[I.t0] * tcols[I.t0];
                tile_add(T0, sm + (int)I.t1 * TSZ);
            } break;
            case VM_TRTRI: {
                const int mm = trows[I.t1];
                if (threadIdx.x == 0) c_fl += (double)mm * mm * mm / 3.0;
                tile_trtri(T0, sm + (int)I.t1 * TSZ, mm);
                if (threadIdx.x == 0) { trows[I.t0] = mm; tcols[I.t0] = mm; }
                __syncthreads();
            } break;
            case VM_ZERO: {
                tile_zero(T0);
                if (threadIdx.x == 0) {
                    trows[I.t0] = dim_eval(I.rows, ranks);
                    tcols[I.t0] = dim_eval(I.cols, ranks);
                }
                __syncthreads();
            } break;
            case VM_GEMM: {
                const double* T1 = sm + (int)I.t1 * TSZ;
                const double* T2 = sm + (int)I.t2 * TSZ;
                const int m = I.ta ? tcols[I.t1] : trows[I.t1];
                const int ka = I.ta ? trows[I.t1] : tcols[I.t1];
                const int kb = I.tb ? tcols[I.t2] : trows[I.t2];
                const int n = I.tb ? trows[I.t2] : tcols[I.t2];
                const int k = max(ka, kb);
                if (I.beta == 0.0) {
                    tile_zero(T0);
                    __syncthreads();
                    if (threadIdx.x == 0) { trows[I.t0] = m; tcols[I.t0] = n; }
                }
                if (threadIdx.x == 0) c_fl += 2.0 * m * n * k;
                if (m > 0 && n > 0 && k > 0)
                    tile_gemm(T0, T1, I.ta != 0, T2, I.tb != 0, m, n, k, I.alpha, I.beta == 0.0 ? 0.0 : I.beta);
                __syncthreads();
            } break;
            case VM_POTRF: {
                if (threadIdx.x == 0) c_fl += (double)trows[I.t0] * trows[I.t0] * trows[I.t0] / 3.0;
                const int f = tile_potrf(T0, trows[I.t0], &s_log);
                if (threadIdx.x == 0) {
                    pool[I.goff] = s_log;
                    if (f) atomicAdd(flags, f);
                }
                __syncthreads();
            } break;
            case VM_TRSM_RLT: {
                if (threadIdx.x == 0) c_fl += (double)trows[I.t0] * tcols[I.t0] * tcols[I.t0];
                tile_trsm_rlt(T0, sm + (int)I.t1 * TSZ, trows[I.t0], tcols[I.t0]);
            } break;
            case VM_TRSM_LN: {
                if (threadIdx.x == 0) c_fl += (double)trows[I.t0] * trows[I.t0] * tcols[I.t0];
                tile_trsm_ln(T0, sm + (int)I.t1 * TSZ, trows[I.t0], tcols[I.t0]);
            } break;
            case VM_TRMM_LN: {
                if (threadIdx.x == 0) c_fl += (double)trows[I.t0] * trows[I.t0] * tcols[I.t0];
                tile_trmm_ln(T0, sm + (int)I.t1 * TSZ, trows[I.t0], tcols[I.t0]);
            } break;
            default:
                break;
        }
    }
    if (threadIdx.x == 0) {
        atomicAdd(ctr + CTR_VM + 0, c_fl);
        atomicAdd(ctr + CTR_VM + 1, c_by);
    }
}

}  // namespace hm

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
// GM_NS-stage cp.async pipeline (zero-filled outside each operand's dims) into
// `stage` (the free tiles 1..2), and accumulated in registers by the FP64 tensor
// cores (warp tile 16 x 32, 4 x 2 warps); T0 is updated once at the end.
struct TermRt {
    const double* a;
    const double* b;
    int32_t lda, ldb, M, N, K, ch0;   // op(A) M x K, op(B) K x N; first chunk index
    int32_t ta, tb;
    int32_t va, vb;                   // operand staged with 16-byte copies (contiguous along M / N, aligned)
    double alpha;
};

// dst == nullptr: T0 += result (smem tile); else dst[r + c ldd] = beta dst + result for
// r < drows, c < dcols (VM_MGEMM_ST: accumulators straight to global memory)
__device__ __forceinline__ void vm_mgemm(double* T0, const VTerm* __restrict__ terms, int nt, const double* pool,
                                         const int* ranks, double* stageA, double* stageB, double& c_fl, double& c_by,
                                         double* dst = nullptr, int64_t ldd = 0, int drows = 0, int dcols = 0,
                                         double beta = 0.0, unsigned long long* stt = nullptr) {
    // staged chunks [k][i] / [k][j]: ld 68 for an operand contiguous along the tile dimension
    // (16-byte copies of element pairs, conflict-free fragment loads), 65 for one contiguous
    // along k (8-byte copies; 65 keeps their stores conflict-free)
    constexpr int SA = GM_BK * 68, SB = GM_BK * 68;
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
        r.va = !v.ta && ((reinterpret_cast<uintptr_t>(r.a) & 15) == 0) && ((v.a_ld & 1) == 0);
        r.vb = v.tb && ((reinterpret_cast<uintptr_t>(r.b) & 15) == 0) && ((v.b_ld & 1) == 0);
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
    static_assert(GM_NS * SA <= TSZ && GM_NS * SB <= TSZ, "stages fit one tile each");
    double* As = stageA;                                 // the two tiles other than T0
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
        double* as = As + (s % GM_NS) * SA;
        double* bs = Bs + (s % GM_NS) * SB;
        if (r.va) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {                // 512 pairs = 64 x 16 / 2
                const int pr = threadIdx.x + e * 256, i = 2 * (pr & 31), k = pr >> 5;
                const int n = (k0 + k < r.K) ? (i + 1 < r.M ? 2 : (i < r.M ? 1 : 0)) : 0;
                cp_async16(as + k * 68 + i, n ? r.a + i + (int64_t)(k0 + k) * r.lda : r.a, 8 * n);
            }
        } else {
            const int la = r.ta ? 65 : 68;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int idx = threadIdx.x + e * 256;     // 1024 = 64 x 16
                int i, k;
                if (r.ta) { k = idx % GM_BK; i = idx / GM_BK; } else { i = idx % 64; k = idx / 64; }
                const bool ok = i < r.M && k0 + k < r.K;
                cp_async8(as + k * la + i,
                          ok ? (r.ta ? r.a + (k0 + k) + (int64_t)i * r.lda : r.a + i + (int64_t)(k0 + k) * r.lda) : r.a, ok);
            }
        }
        if (r.vb) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int pr = threadIdx.x + e * 256, j = 2 * (pr & 31), kb = pr >> 5;
                const int n = (k0 + kb < r.K) ? (j + 1 < r.N ? 2 : (j < r.N ? 1 : 0)) : 0;
                cp_async16(bs + kb * 68 + j, n ? r.b + j + (int64_t)(k0 + kb) * r.ldb : r.b, 8 * n);
            }
        } else {
            const int lb = r.tb ? 68 : 65;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int idx = threadIdx.x + e * 256;
                int j, kb;
                if (r.tb) { j = idx % 64; kb = idx / 64; } else { kb = idx % GM_BK; j = idx / GM_BK; }
                const bool okb = j < r.N && k0 + kb < r.K;
                cp_async8(bs + kb * lb + j,
                          okb ? (r.tb ? r.b + j + (int64_t)(k0 + kb) * r.ldb : r.b + (k0 + kb) + (int64_t)j * r.ldb) : r.b,
                          okb);
            }
        }
        ++ik;
    };
    int ct = 0, ck = 0;                                  // compute cursor
    auto compute = [&](int s) {
        while (ct < nt && ck >= (tr[ct].K + GM_BK - 1) / GM_BK) { ++ct; ck = 0; }
        const double al = tr[ct].alpha;
        const int la = tr[ct].ta ? 65 : 68, lb = tr[ct].tb ? 68 : 65;
        // fragments outside this term's op(A) rows / op(B) columns get zeros from it: skip
        // their DMMAs (warp-uniform; low-rank factors are often much narrower than 64)
        const int am = tr[ct].M - wm, bn = tr[ct].N - wn, kr = tr[ct].K - ck * GM_BK;
        ++ck;
        if (am <= 0 || bn <= 0) return;
        const double* as = As + (s % GM_NS) * SA;
        const double* bs = Bs + (s % GM_NS) * SB;
#pragma unroll
        for (int kk = 0; kk < GM_BK; kk += 4) {
            if (kk >= kr) break;
            double af[2], bf[4];
#pragma unroll
            for (int a = 0; a < 2; ++a) af[a] = al * as[(kk + t4) * la + wm + a * 8 + g];
#pragma unroll
            for (int b = 0; b < 4; ++b) bf[b] = bs[(kk + t4) * lb + wn + b * 8 + g];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (a * 8 < am && b * 8 < bn) dmma_884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
    };
    if (nch <= GM_NS) {
        // short sums (the latency-bound tasks on the Cholesky's critical path): every chunk
        // in flight at once, a single wait
        for (int s = 0; s < nch; ++s) issue(s);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        for (int s = 0; s < nch; ++s) compute(s);
    } else {
#pragma unroll
        for (int s = 0; s < GM_NS - 1; ++s) {
            issue(s);
            cp_async_commit();
        }
        for (int s = 0; s < nch; ++s) {
            cp_async_wait<GM_NS - 2>();
            __syncthreads();
            if (s + GM_NS - 1 < nch) issue(s + GM_NS - 1);
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
                const int o1 = (I.t0 == 0) ? 1 : 0, o2 = (I.t0 == 2) ? 1 : 2;   // staging: the other tiles
                vm_mgemm(T0, terms + I.goff, I.ld, pool, ranks, sm + o1 * TSZ, sm + o2 * TSZ, c_fl, c_by);
            } break;
            case VM_MGEMM_ST: {
                const int o1 = (I.t0 == 0) ? 1 : 0, o2 = (I.t0 == 2) ? 1 : 2;
                const int r = dim_eval(I.rows, ranks), c = dim_eval(I.cols, ranks);
                vm_mgemm(T0, terms + I.pad2, I.t1, pool, ranks, sm + o1 * TSZ, sm + o2 * TSZ, c_fl, c_by, pool + I.goff,
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

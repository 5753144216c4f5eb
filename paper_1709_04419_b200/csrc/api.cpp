// C-ABI entry points: errors, geometry, dense check path, Matern test hook.
// (The H-matrix entry points live in hmatrix_api.cpp.)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/hmlik.h"
#include "api_util.h"
#include "common.h"
#include "dense.h"
#include "plan.h"
#include "sched.h"
#include "tree.h"

struct hm_tree_s {
    hm::Tree T;
};

namespace hm {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int translate_exception() {
    try {
        throw;
    } catch (const CudaError& e) {
        return set_error(HM_ERR_CUDA, std::string("CUDA error '") + cudaGetErrorString(e.err) + "' in " + e.expr +
                                          " (" + e.file + ":" + std::to_string(e.line) + ")");
    } catch (const ApiError& e) {
        return set_error(e.code, e.what());
    } catch (const std::invalid_argument& e) {
        return set_error(HM_ERR_ARG, e.what());
    } catch (const std::bad_alloc&) {
        return set_error(HM_ERR_OOM, "host allocation failed");
    } catch (const std::exception& e) {
        return set_error(HM_ERR_STATE, e.what());
    } catch (...) {
        return set_error(HM_ERR_STATE, "unknown exception");
    }
}

void check_theta(const hm_theta& th) {
    if (!(th.sigma2 > 0 && th.ell > 0 && th.nu > 0) || !std::isfinite(th.sigma2) || !std::isfinite(th.ell) ||
        !std::isfinite(th.nu))
        throw ApiError(HM_ERR_ARG, "theta must be finite with sigma2, ell, nu > 0");
}

DevBuf::~DevBuf() {
    if (p) cudaFree(p);
}
void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

void DevBuf::alloc(size_t b) {
    if (b <= bytes && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (b == 0) return;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw ApiError(HM_ERR_OOM, std::string("cudaMalloc(") + std::to_string(b) + ") failed: " + cudaGetErrorString(e));
    }
    bytes = b;
}

DeviceGuard::DeviceGuard(int dev) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw ApiError(HM_ERR_CUDA, "no CUDA device available (the library has no CPU path)");
    }
    if (dev < 0 || dev >= n) throw ApiError(HM_ERR_ARG, "invalid CUDA device ordinal");
    HM_CUDA_TRY(cudaGetDevice(&prev));
    HM_CUDA_TRY(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
}

}  // namespace hm

using namespace hm;

extern "C" {

const char* hm_last_error(void) { return g_last_error.c_str(); }
const char* hm_version(void) { return "hmlik 0.1 (sm_100a)"; }

int hm_tree_build(const double* locs_host, int64_t n, int32_t leaf, double eta, hm_tree* out) {
    try {
        if (!out || !locs_host) throw ApiError(HM_ERR_ARG, "null pointer");
        auto* t = new hm_tree_s();
        try {
            build_tree(locs_host, n, leaf, eta, t->T);
        } catch (...) {
            delete t;
            throw;
        }
        *out = t;
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_tree_free(hm_tree t) {
    delete t;
    return HM_OK;
}

int hm_tree_counts(hm_tree t, int64_t counts[6]) {
    if (!t || !counts) return set_error(HM_ERR_ARG, "null pointer");
    const Tree& T = t->T;
    counts[0] = T.n;
    counts[1] = (int64_t)T.clusters.size();
    counts[2] = T.n_leaf_clusters;
    counts[3] = T.depth;
    counts[4] = (int64_t)T.full_blocks.size() / 6;
    int64_t adm = 0;
    for (size_t i = 0; i < T.full_blocks.size(); i += 6) adm += T.full_blocks[i + 5];
    counts[5] = adm;
    return HM_OK;
}

int hm_tree_perm(hm_tree t, int64_t* perm_host) {
    if (!t || !perm_host) return set_error(HM_ERR_ARG, "null pointer");
    std::memcpy(perm_host, t->T.perm.data(), sizeof(int64_t) * t->T.perm.size());
    return HM_OK;
}

int hm_tree_clusters(hm_tree t, int64_t* out) {
    if (!t || !out) return set_error(HM_ERR_ARG, "null pointer");
    // pre-order == storage order
    size_t k = 0;
    for (const auto& c : t->T.clusters) {
        out[k++] = c.lo;
        out[k++] = c.hi;
        out[k++] = c.level;
        out[k++] = c.leaf() ? 1 : 0;
    }
    return HM_OK;
}

int hm_tree_blocks(hm_tree t, int64_t* out) {
    if (!t || !out) return set_error(HM_ERR_ARG, "null pointer");
    std::memcpy(out, t->T.full_blocks.data(), sizeof(int64_t) * t->T.full_blocks.size());
    return HM_OK;
}

int hm_plan_dump(hm_tree t, int32_t kmax, const char* path, double summary[8]) {
    try {
        if (!t) throw ApiError(HM_ERR_ARG, "null tree");
        if (kmax <= 0) kmax = 160;
        Plan P;
        build_plan(t->T, kmax, P);
        // the executor's ready-queue schedule of every phase, with its host replay
        // self-check (sched.cpp): validated here without a GPU
        for (const Phase* ph : {&P.recompress, &P.chol, &P.solve, &P.lmul}) {
            Sched sc;
            build_sched(*ph, sc);
        }
        if (summary) {
            summary[0] = (double)P.pool_total;
            summary[1] = P.n_slots;
            summary[2] = (double)P.chol.vt.size();
            summary[3] = (double)P.chol.tt.size();
            summary[4] = P.chol.nwaves;
            summary[5] = (double)P.chol.n_launches();
            summary[6] = P.solve.nwaves;
            summary[7] = (double)(P.solve.vt.size() + P.solve.tt.size());
        }
        if (path) {
            FILE* f = std::fopen(path, "wb");
            if (!f) throw ApiError(HM_ERR_ARG, std::string("cannot open ") + path);
            auto put = [&](const void* p, int64_t count, int64_t size) {
                std::fwrite(&count, 8, 1, f);
                std::fwrite(&size, 8, 1, f);
                if (count) std::fwrite(p, (size_t)size, (size_t)count, f);
            };
            int64_t hdr[8] = {P.pool_total, P.n_slots, P.logd_off, P.z_off, P.zw, t->T.n, P.n_leaves, P.z_slot};
            put(hdr, 8, 8);
            put(P.dgen.data(), (int64_t)P.dgen.size(), sizeof(DenseGenTask));
            put(P.aca.data(), (int64_t)P.aca.size(), sizeof(AcaTask));
            for (const Phase* ph : {&P.recompress, &P.chol, &P.solve, &P.lmul}) {
                put(ph->ins.data(), (int64_t)ph->ins.size(), sizeof(VIns));
                put(ph->vt.data(), (int64_t)ph->vt.size(), sizeof(VTask));
                put(ph->tt.data(), (int64_t)ph->tt.size(), sizeof(TTask));
                put(ph->tp.data(), (int64_t)ph->tp.size(), sizeof(TPiece));
                put(ph->v_wave_begin.data(), (int64_t)ph->v_wave_begin.size(), 4);
                put(ph->t_wave_begin.data(), (int64_t)ph->t_wave_begin.size(), 4);
                put(ph->xt.data(), (int64_t)ph->xt.size(), sizeof(XTask));
                put(ph->xdeps.data(), (int64_t)ph->xdeps.size(), 4);
                put(ph->terms.data(), (int64_t)ph->terms.size(), sizeof(VTerm));
            }
            std::fclose(f);
        }
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_dense_loglik(const double* locs, int32_t locs_on_device, int64_t n, hm_theta theta, const double* Z,
                    int32_t z_on_device, int32_t k, int32_t device, void* stream, double* out_host) {
    try {
        if (!locs || !Z || !out_host) throw ApiError(HM_ERR_ARG, "null pointer");
        if (n < 1 || k < 1) throw ApiError(HM_ERR_ARG, "n >= 1 and k >= 1 required");
        if (n > HM_DENSE_NMAX) throw ApiError(HM_ERR_TOO_LARGE, "dense check path is limited to n <= " + std::to_string(HM_DENSE_NMAX));
        check_theta(theta);
        DeviceGuard dg(device);
        cudaStream_t st = (cudaStream_t)stream;
        MaternParams p;
        matern_setup(theta.sigma2, theta.ell, theta.nu, p);
        DevBuf A, P, Zd, logd, fail, out;
        A.alloc(sizeof(double) * (size_t)n * (size_t)n);
        P.alloc(sizeof(double) * 2 * n);
        Zd.alloc(sizeof(double) * (size_t)n * k);
        const int64_t nblk = (n + 63) / 64;
        logd.alloc(sizeof(double) * nblk);
        fail.alloc(sizeof(int));
        out.alloc(sizeof(double) * 3 * k);
        HM_CUDA_TRY(cudaMemcpyAsync(P.p, locs, sizeof(double) * 2 * n,
                                    locs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        HM_CUDA_TRY(cudaMemcpyAsync(Zd.p, Z, sizeof(double) * (size_t)n * k,
                                    z_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        dense_loglik_device((double*)P.p, n, p, (double*)Zd.p, k, (double*)A.p, (double*)logd.p, (int*)fail.p,
                            (double*)out.p, st);
        int hfail = 0;
        HM_CUDA_TRY(cudaMemcpyAsync(&hfail, fail.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        HM_CUDA_TRY(cudaMemcpyAsync(out_host, out.p, sizeof(double) * 3 * k, cudaMemcpyDeviceToHost, st));
        HM_CUDA_TRY(cudaStreamSynchronize(st));
        if (hfail) throw ApiError(HM_ERR_NOT_SPD, "dense Cholesky: non-positive pivot");
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

int hm_matern_block(const double* a_host, int64_t ni, const double* b_host, int64_t nj, hm_theta theta, int32_t device,
                    double* out_host) {
    try {
        if (!a_host || !b_host || !out_host) throw ApiError(HM_ERR_ARG, "null pointer");
        if (ni < 0 || nj < 0) throw ApiError(HM_ERR_ARG, "negative size");
        check_theta(theta);
        DeviceGuard dg(device);
        MaternParams p;
        matern_setup(theta.sigma2, theta.ell, theta.nu, p);
        DevBuf A, B, O;
        A.alloc(sizeof(double) * 2 * (ni + 1));
        B.alloc(sizeof(double) * 2 * (nj + 1));
        O.alloc(sizeof(double) * (ni * nj + 1));
        HM_CUDA_TRY(cudaMemcpy(A.p, a_host, sizeof(double) * 2 * ni, cudaMemcpyHostToDevice));
        HM_CUDA_TRY(cudaMemcpy(B.p, b_host, sizeof(double) * 2 * nj, cudaMemcpyHostToDevice));
        matern_block_device((double*)A.p, ni, (double*)B.p, nj, p, (double*)O.p, 0);
        HM_CUDA_TRY(cudaMemcpy(out_host, O.p, sizeof(double) * ni * nj, cudaMemcpyDeviceToHost));
        return HM_OK;
    } catch (...) {
        return translate_exception();
    }
}

}  // extern "C"

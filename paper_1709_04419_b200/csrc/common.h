// Shared host/device declarations for the hmlik library (no torch types).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hm {

// theta-derived constants for the device Matern kernel, Eq. (2).
// Filled on the host by matern_setup(); `kind` selects a closed form for the
// half-integer orders (l.188: nu = 1/2 is the exponential model).
struct MaternParams {
    double sigma2, ell, nu;
    double coef;          // sigma2 / (2^(nu-1) Gamma(nu))
    int32_t kind;         // 0 general Bessel path, 1: nu=1/2, 2: nu=3/2, 3: nu=5/2
    int32_t nl;           // nu = nl + mu, mu in [-1/2, 1/2)
    double mu;
    double fact;          // pi mu / sin(pi mu)    (Temme series)
    double gam1, gam2;    // (1/G(1-mu) - 1/G(1+mu))/(2mu), (1/G(1-mu) + 1/G(1+mu))/2
    double gampl, gammi;  // 1/G(1+mu), 1/G(1-mu)
};

void matern_setup(double sigma2, double ell, double nu, MaternParams& p);

}  // namespace hm

#define HM_CUDA_TRY(expr)                                                         \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) throw hm::CudaError(_e, #expr, __FILE__, __LINE__); \
    } while (0)

namespace hm {
struct CudaError {
    cudaError_t err;
    const char* expr;
    const char* file;
    int line;
    CudaError(cudaError_t e, const char* x, const char* f, int l) : err(e), expr(x), file(f), line(l) {}
};
}  // namespace hm

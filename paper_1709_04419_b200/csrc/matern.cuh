// Device Matern covariance (Eq. 2, l.183-188) with a device K_nu.
//
// K_nu(x), fractional order nu = n + mu with |mu| <= 1/2 (n = nl):
//  * x <= 2: Temme's power series for the pair K_mu, K_{mu+1}
//      N. M. Temme, "On the numerical evaluation of the modified Bessel function
//      of the third kind", J. Comput. Phys. 19 (1975) 324-337, eqs. (2.5)-(2.9);
//  * x > 2: the continued fraction for K_{mu+1} / K_mu evaluated by Steed's
//    method, normalised by Temme's companion series (the "CF2" of
//      I. J. Thompson and A. R. Barnett, "Modified Bessel functions I_nu(z) and
//      K_nu(z) of real order and complex argument, to selected accuracy",
//      Comput. Phys. Commun. 47 (1987) 245-257, sec. 3; A. R. Barnett et al.,
//      Comput. Phys. Commun. 8 (1974) 377-395 for Steed's algorithm);
//  * then the three-term recurrence K_{a+1} = K_{a-1} + (2a/x) K_a (DLMF 10.29.1)
//    upward to order nu (stable for K).
// The mu-only Gamma-function constants are precomputed on the host
// (matern_setup, matern_host.cpp).  This is independent of the oracle's
// trapezoidal quadrature of the integral representation (oracle/matern.py).
#pragma once
#include "common.h"

namespace hm {

struct KPair {   // K_mu(x), K_{mu+1}(x)
    double k0, k1;
};

// Temme's series, x <= 2:  with c_k = (x^2/4)^k / k!,
//   K_mu = sum_k c_k f_k,   K_{mu+1} = (2/x) sum_k c_k (p_k - k f_k),
//   f_k = (k f_{k-1} + p_{k-1} + q_{k-1}) / (k^2 - mu^2),  p_k = p_{k-1} / (k - mu),  q_k = q_{k-1} / (k + mu),
//   f_0 = (pi mu / sin pi mu) [cosh(s) G1 + (sinh(s)/s) ln(2/x) G2],  s = mu ln(2/x),
//   p_0 = (x/2)^-mu Gamma(1+mu) / 2,  q_0 = (x/2)^mu Gamma(1-mu) / 2.
__device__ __forceinline__ KPair temme_series(double x, const MaternParams& p) {
    const double mu = p.mu;
    const double lg = -log(0.5 * x);                 // ln(2/x)
    const double s = mu * lg;
    const double sinhc = (fabs(s) < 1e-300) ? 1.0 : sinh(s) / s;
    const double es = exp(s);                        // (x/2)^-mu
    double f = p.fact * (p.gam1 * cosh(s) + p.gam2 * sinhc * lg);
    double pk = 0.5 * es / p.gampl;
    double qk = 0.5 / (es * p.gammi);
    const double x2q = 0.25 * x * x;
    double ck = 1.0;
    double sum0 = f, sum1 = pk;
    for (int k = 1; k < 200; ++k) {
        const double dk = (double)k;
        f = (dk * f + pk + qk) / (dk * dk - mu * mu);
        ck *= x2q / dk;
        pk /= dk - mu;
        qk /= dk + mu;
        const double t0 = ck * f;
        sum0 += t0;
        sum1 += ck * (pk - dk * f);
        if (fabs(t0) < 1e-16 * fabs(sum0)) break;
    }
    return KPair{sum0, sum1 * (2.0 / x)};
}

// x > 2: the ratio K_{mu+1}/K_mu = (mu + x + 1/2 - a_1 r) / x with r the continued
// fraction r = 1 / (b_1 + a_2 / (b_2 + ...)), b_k = 2 (x + k), a_k = -((k - 1/2)^2 - mu^2),
// summed term by term by Steed's method; the normalisation comes from the series
// S = 1 + sum_k Q_k (t_k) of the same recursion (Thompson & Barnett), so that
// K_mu = sqrt(pi / 2x) e^-x / S.
__device__ __forceinline__ KPair steed_cf2(double x, const MaternParams& p) {
    const double mu = p.mu;
    const double a1 = 0.25 - mu * mu;
    double bk = 2.0 * (1.0 + x);
    double dk = 1.0 / bk;
    double term = dk, r = dk;                        // Steed: r = sum of the convergent increments
    double qprev = 0.0, qcur = 1.0;                  // Q_{k-1}, Q_k of the normalisation recursion
    double ak = -a1;
    double ck = a1, qsum = a1;
    double snorm = 1.0 + qsum * term;
    for (int k = 2; k < 1000; ++k) {
        ak -= 2.0 * (double)(k - 1);
        ck = -ak * ck / (double)k;
        const double qnext = (qprev - bk * qcur) / ak;
        qprev = qcur;
        qcur = qnext;
        qsum += ck * qnext;
        bk += 2.0;
        dk = 1.0 / (bk + ak * dk);
        term = (bk * dk - 1.0) * term;
        r += term;
        const double ds = qsum * term;
        snorm += ds;
        if (fabs(ds) < 1e-16 * fabs(snorm)) break;
    }
    const double k0 = sqrt(3.14159265358979323846 / (2.0 * x)) * exp(-x) / snorm;
    return KPair{k0, k0 * (mu + x + 0.5 - a1 * r) / x};
}

__device__ __forceinline__ double bessel_k_dev(double x, const MaternParams& p) {
    KPair k = (x <= 2.0) ? temme_series(x, p) : steed_cf2(x, p);
    for (int i = 1; i <= p.nl; ++i) {               // K_{a+1} = K_{a-1} + (2a/x) K_a, a = mu + i
        const double next = (p.mu + (double)i) * (2.0 / x) * k.k1 + k.k0;
        k.k0 = k.k1;
        k.k1 = next;
    }
    return k.k0;
}

// C(h; theta), h >= 0.
__device__ __forceinline__ double matern_dev(double h, const MaternParams& p) {
    if (h == 0.0) return p.sigma2;
    const double x = h / p.ell;
    switch (p.kind) {
        case 1: return p.sigma2 * exp(-x);
        case 2: return p.sigma2 * (1.0 + x) * exp(-x);
        case 3: return p.sigma2 * (1.0 + x + x * x / 3.0) * exp(-x);
        default: break;
    }
    if (x > 740.0) return 0.0;
    return p.coef * pow(x, p.nu) * bessel_k_dev(x, p);
}

__device__ __forceinline__ double dist2d(double ax, double ay, double bx, double by) {
    const double dx = ax - bx, dy = ay - by;
    return sqrt(dx * dx + dy * dy);
}

}  // namespace hm

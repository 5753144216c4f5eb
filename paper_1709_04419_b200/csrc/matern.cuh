// Device Matern covariance (Eq. 2, l.183-188) with a device K_nu.
//
// K_nu(x) for fractional order: nu = nl + mu with |mu| <= 1/2; K_mu and
// K_{mu+1} from Temme's series for x < 2 and from Steed's continued fraction
// (CF2, Thompson-Barnett) for x >= 2, then forward recurrence
// K_{a+1} = K_{a-1} + (2a/x) K_a up to order nu.  mu-only constants (Gamma
// function combinations) are precomputed on the host (matern_setup).  This is
// an independent algorithm from the oracle's quadrature of the integral
// representation.
#pragma once
#include "common.h"

namespace hm {

__device__ __forceinline__ double bessel_k_dev(double x, const MaternParams& p) {
    const double EPS = 1.0e-16;
    const double mu = p.mu;
    double rkmu, rk1;
    if (x < 2.0) {
        // Temme's series
        const double x2 = 0.5 * x;
        const double d = -log(x2);
        const double e = mu * d;
        const double fact2 = (fabs(e) < 1e-300) ? 1.0 : sinh(e) / e;
        double ff = p.fact * (p.gam1 * cosh(e) + p.gam2 * fact2 * d);
        double sum = ff;
        const double ee = exp(e);
        double pp = 0.5 * ee / p.gampl;
        double qq = 0.5 / (ee * p.gammi);
        double c = 1.0;
        const double dd = x2 * x2;
        double sum1 = pp;
        for (int i = 1; i < 200; ++i) {
            const double fi = (double)i;
            ff = (fi * ff + pp + qq) / (fi * fi - mu * mu);
            c *= dd / fi;
            pp /= (fi - mu);
            qq /= (fi + mu);
            const double del = c * ff;
            sum += del;
            const double del1 = c * (pp - fi * ff);
            sum1 += del1;
            if (fabs(del) < fabs(sum) * EPS) break;
        }
        rkmu = sum;
        rk1 = sum1 * (2.0 / x);
    } else {
        // Steed's continued fraction CF2
        double b = 2.0 * (1.0 + x);
        double d = 1.0 / b;
        double h = d, delh = d;
        double q1 = 0.0, q2 = 1.0;
        const double a1 = 0.25 - mu * mu;
        double q = a1, c = a1;
        double a = -a1;
        double s = 1.0 + q * delh;
        for (int i = 2; i < 1000; ++i) {
            a -= 2.0 * (double)(i - 1);
            c = -a * c / (double)i;
            const double qnew = (q1 - b * q2) / a;
            q1 = q2;
            q2 = qnew;
            q += c * qnew;
            b += 2.0;
            d = 1.0 / (b + a * d);
            delh = (b * d - 1.0) * delh;
            h += delh;
            const double dels = q * delh;
            s += dels;
            if (fabs(dels / s) < EPS) break;
        }
        rkmu = sqrt(3.14159265358979323846 / (2.0 * x)) * exp(-x) / s;
        rk1 = rkmu * (mu + x + 0.5 - a1 * h) / x;
    }
    for (int i = 1; i <= p.nl; ++i) {
        const double t = (mu + (double)i) * (2.0 / x) * rk1 + rkmu;
        rkmu = rk1;
        rk1 = t;
    }
    return rkmu;
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

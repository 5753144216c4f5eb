// Host setup of the theta-dependent constants of the device Matern kernel
// (Eq. 2, l.183-188).  See matern.cuh for the device algorithm and its
// sources (Temme 1975; Thompson & Barnett 1987): the order split nu = n + mu and
// Temme's Gamma-function combinations
//   G1(mu) = (1/Gamma(1-mu) - 1/Gamma(1+mu)) / (2 mu),  G2(mu) = (1/Gamma(1-mu) + 1/Gamma(1+mu)) / 2,
// evaluated from the Taylor series of 1/Gamma (accurate also as mu -> 0).
#include <cmath>

#include "common.h"

namespace hm {

// Taylor coefficients of 1/Gamma(z) = sum_{k>=1} c_k z^k (Abramowitz & Stegun 6.1.34),
// so 1/Gamma(1+z) = sum_{k>=1} c_k z^{k-1}.  Converges to < 1e-16 for |z| <= 1/2.
static const double kRecipGamma[26] = {
    1.0,                 0.5772156649015329,  -0.6558780715202538, -0.0420026350340952,
    0.1665386113822915,  -0.0421977345555443, -0.0096219715278770, 0.0072189432466630,
    -0.0011651675918591, -0.0002152416741149, 0.0001280502823882,  -0.0000201348547807,
    -0.0000012504934821, 0.0000011330272320,  -0.0000002056338417, 0.0000000061160950,
    0.0000000050020075,  -0.0000000011812746, 0.0000000001043427,  0.0000000000077823,
    -0.0000000000036968, 0.0000000000005100,  -0.0000000000000206, -0.0000000000000054,
    0.0000000000000014,  0.0000000000000001};

void matern_setup(double sigma2, double ell, double nu, MaternParams& p) {
    p.sigma2 = sigma2;
    p.ell = ell;
    p.nu = nu;
    p.coef = sigma2 / (std::pow(2.0, nu - 1.0) * std::tgamma(nu));
    p.kind = 0;
    if (nu == 0.5) p.kind = 1;
    else if (nu == 1.5) p.kind = 2;
    else if (nu == 2.5) p.kind = 3;
    p.nl = (int32_t)(nu + 0.5);
    p.mu = nu - (double)p.nl;
    const double mu = p.mu;
    const double pimu = M_PI * mu;
    p.fact = (std::fabs(pimu) < 1e-300) ? 1.0 : pimu / std::sin(pimu);
    double gampl = 0.0, gammi = 0.0, gam1 = 0.0, gam2 = 0.0;
    double pw = 1.0, pwm = 1.0;  // mu^k, (-mu)^k
    for (int k = 0; k < 26; ++k) {
        gampl += kRecipGamma[k] * pw;
        gammi += kRecipGamma[k] * pwm;
        pw *= mu;
        pwm *= -mu;
    }
    // gam1 = (1/G(1-mu) - 1/G(1+mu)) / (2 mu) = -(c_2 + c_4 mu^2 + c_6 mu^4 + ...)
    // gam2 = (1/G(1-mu) + 1/G(1+mu)) / 2    =   c_1 + c_3 mu^2 + c_5 mu^4 + ...
    double m2 = 1.0;
    for (int k = 1; k < 26; k += 2) {
        gam1 -= kRecipGamma[k] * m2;
        m2 *= mu * mu;
    }
    m2 = 1.0;
    for (int k = 0; k < 26; k += 2) {
        gam2 += kRecipGamma[k] * m2;
        m2 *= mu * mu;
    }
    p.gampl = gampl;
    p.gammi = gammi;
    p.gam1 = gam1;
    p.gam2 = gam2;
}

}  // namespace hm

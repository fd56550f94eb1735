/*
 * e_float certificate of arXiv 2507.09165, Eq. (comp:error-approx):
 *
 *     e_float(f) = max_{x in S_float} |f(x) - relu(x)|,
 *     S_float = every float32 in [-1, 1]  (2,130,706,433 values),
 *     f(x) = 1/2 x (1 + s(x)),  s = f_T o ... o f_1   (Eq. comp:fstar).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain loops in double,
 * OpenMP over bit patterns.  s is odd, so |f(x) - relu(x)| = 1/2 |x| |1 - s(|x|)|
 * is even in x and the maximum over [-1,1] equals the maximum over [0,1]:
 * bit patterns 0x00000000 .. 0x3F800000.
 *
 * Also: the sign error max_{x in [eps,1] float32} |s(x) - 1| (Eq. comp:minimax-sign,
 * P:L502-506 restricted to the positive half by oddness).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double chain(double x, int T, const int* ncoef, const double* coeffs, const double* kappas) {
    const double* c = coeffs;
    for (int t = 0; t < T; ++t) {
        double x2 = x * x, pw = x, acc = 0.0;
        for (int j = 0; j < ncoef[t]; ++j) {   /* sum_j c_j x^{2j+1} */
            acc += c[j] * pw;
            pw *= x2;
        }
        x = acc;
        if (kappas) x *= kappas[t];
        c += ncoef[t];
    }
    return x;
}

static float bits_to_float(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* max over float32 x in [0,1] of 1/2 x |1 - s(x)|; returns the ReLU-convention error. */
double certify_relu_err(int T, const int* ncoef, const double* coeffs, const double* kappas,
                        double* argmax_out, long long* count_out) {
    const uint32_t last = 0x3F800000u;   /* 1.0f */
    double best = -1.0, best_x = 0.0;
#pragma omp parallel
    {
        double lb = -1.0, lx = 0.0;
#pragma omp for schedule(static)
        for (long long u = 0; u <= (long long)last; ++u) {
            double x = (double)bits_to_float((uint32_t)u);
            double e = 0.5 * x * fabs(1.0 - chain(x, T, ncoef, coeffs, kappas));
            if (e > lb) { lb = e; lx = x; }
        }
#pragma omp critical
        {
            if (lb > best || (lb == best && lx < best_x)) { best = lb; best_x = lx; }
        }
    }
    if (argmax_out) *argmax_out = best_x;
    if (count_out) *count_out = 2LL * (long long)last + 1LL;   /* |S_float| incl. +-0 once */
    return best;
}

/* max over float32 x in [eps,1] of |s(x) - 1|. */
double certify_sign_err(int T, const int* ncoef, const double* coeffs, const double* kappas,
                        double eps, double* argmax_out) {
    float fe = (float)eps;
    if ((double)fe < eps) fe = nextafterf(fe, 2.0f);   /* first float32 >= eps */
    uint32_t first; memcpy(&first, &fe, 4);
    const uint32_t last = 0x3F800000u;
    double best = -1.0, best_x = 0.0;
#pragma omp parallel
    {
        double lb = -1.0, lx = 0.0;
#pragma omp for schedule(static)
        for (long long u = first; u <= (long long)last; ++u) {
            double x = (double)bits_to_float((uint32_t)u);
            double e = fabs(chain(x, T, ncoef, coeffs, kappas) - 1.0);
            if (e > lb) { lb = e; lx = x; }
        }
#pragma omp critical
        {
            if (lb > best || (lb == best && lx < best_x)) { best = lb; best_x = lx; }
        }
    }
    if (argmax_out) *argmax_out = best_x;
    return best;
}

int certify_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * c_abi_example.c -- a plain C99 user of the C ABI (include/cpa_svt.h), no CUDA headers, no
 * Python: one dense fp64 shrinkage through cpa_svt_apply_host on HOST buffers, checked
 * element by element against the closed form of Algorithm 1.
 *
 *   gcc -std=c99 -I include examples/c_abi_example.c -L paper_1705_07112_b200 -lcpasvt \
 *       -Wl,-rpath,$PWD/paper_1705_07112_b200 -lm -o c_abi_example
 *   ./c_abi_example [m n K T]
 *
 * Input: X = P D Q, a rectangular diagonal D = diag(d_1..d_s) (s = min(m, n)) with rows and
 * columns permuted and signs flipped (P, Q signed permutations: exact in fp64).  Its Gram is
 * P D^2 P^T (left) or Q^T D^2 Q (right), so for ANY polynomial H_hat the shrinkage is
 *     Y = P D H_hat(D^2) Q      (G(B) = B H(B^T B) = H(B B^T) B),
 * i.e. Y keeps X's support with Y_ij = X_ij H_hat(d^2), d = |X_ij|, where
 *     H_hat(x) = c_0/2 + sum_{k=1}^{K-1} c_k T_k(2 x / Lambda - 1)
 * is evaluated here in scalar fp64 by the three-term recurrence T_k = 2 t T_{k-1} - T_{k-2}
 * (PAPER.md:368), with the library's Lambda (returned through want_lambda) and its host
 * coefficient routine cpa_svt_coeffs.  Prints one line
 *     side=<left|right> form=<f> lambda_max=<L> rel_fro=<e> max_abs=<a>
 * and exits 0 iff rel_fro <= 1e-10 (the fp64 bar of BASELINE.json's north star).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "cpa_svt.h"

/* small counter-based generator (splitmix64): the permutations, signs and diagonal */
static uint64_t mix(uint64_t *s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static void shuffle(int64_t *p, int64_t n, uint64_t *st) {
  int64_t i;
  for (i = 0; i < n; ++i) p[i] = i;
  for (i = n - 1; i > 0; --i) {
    const int64_t j = (int64_t)(mix(st) % (uint64_t)(i + 1));
    const int64_t t = p[i];
    p[i] = p[j];
    p[j] = t;
  }
}

static double h_hat(const double *c, int K, double x, double lambda_max) {
  const double t = 2.0 * x / lambda_max - 1.0;
  double tm2 = 1.0, tm1 = t, acc = 0.5 * c[0] + (K > 1 ? c[1] * t : 0.0);
  int k;
  for (k = 2; k < K; ++k) {
    const double tk = 2.0 * t * tm1 - tm2;
    acc += c[k] * tk;
    tm2 = tm1;
    tm1 = tk;
  }
  return acc;
}

#define CHECK(call)                                                                     \
  do {                                                                                  \
    cpa_svt_status st_ = (call);                                                        \
    if (st_ != CPA_SVT_OK) {                                                            \
      fprintf(stderr, "%s failed: %s (%s)\n", #call, cpa_svt_status_string(st_),        \
              h ? cpa_svt_last_error(h) : "");                                          \
      return 2;                                                                         \
    }                                                                                   \
  } while (0)

int main(int argc, char **argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 300, n = argc > 2 ? atoll(argv[2]) : 500;
  const int K = argc > 3 ? atoi(argv[3]) : 30, T = argc > 4 ? atoi(argv[4]) : 300;
  const int64_t s = m < n ? m : n;
  cpa_svt_handle *h = NULL;
  double *X = calloc((size_t)(m * n), sizeof(double)), *Y = calloc((size_t)(m * n), sizeof(double));
  double *c = malloc((size_t)K * sizeof(double));
  int64_t *pr = malloc((size_t)m * sizeof(int64_t)), *pc = malloc((size_t)n * sizeof(int64_t));
  uint64_t seed = 20170519ull;
  double num = 0.0, den = 0.0, max_abs = 0.0;
  int64_t i, j;
  cpa_svt_kernel kern = {CPA_SVT_SOFT, 0, 1.0, 0.0, 0.0, 0.0};   /* soft, tau = 1 (absolute) */
  cpa_svt_lambda lam = {T, 1, 1.01, 0.0, 0.0};
  cpa_svt_info info;
  if (!X || !Y || !c || !pr || !pc || s < 1 || K < 2) return 3;

  /* X = P D Q: d_i spread over [0.25, 3] (below and above tau), random signs */
  shuffle(pr, m, &seed);
  shuffle(pc, n, &seed);
  for (i = 0; i < s; ++i) {
    const double d = 0.25 + 2.75 * (double)i / (double)(s > 1 ? s - 1 : 1);
    X[pr[i] * n + pc[i]] = (mix(&seed) & 1) ? -d : d;
  }

  CHECK(cpa_svt_init(&h, 0, NULL, NULL, 0, 1));
  CHECK(cpa_svt_apply_host(h, CPA_SVT_F64, CPA_SVT_MATH_NATIVE, m, n, X, Y, &kern, K, &lam, &info));
  CHECK(cpa_svt_coeffs(&kern, K, lam.lambda_max, sqrt(lam.lambda_hat), c));

  /* every element: on X's support Y_ij = X_ij H_hat(X_ij^2), elsewhere exactly 0 in exact
     arithmetic (the library's products of the zero entries round to at most ~1e-16 of the rest) */
  for (i = 0; i < m; ++i)
    for (j = 0; j < n; ++j) {
      const double x = X[i * n + j];
      const double want = x != 0.0 ? x * h_hat(c, K, x * x, lam.lambda_max) : 0.0;
      const double e = Y[i * n + j] - want;
      num += e * e;
      den += want * want;
      if (fabs(e) > max_abs) max_abs = fabs(e);
    }
  {
    const double rel = sqrt(num / (den > 0.0 ? den : 1.0));
    printf("side=%s form=%d lambda_max=%.17g rel_fro=%.3e max_abs=%.3e\n", info.side ? "right" : "left",
           (int)info.form, lam.lambda_max, rel, max_abs);
    CHECK(cpa_svt_free(h));
    free(X);
    free(Y);
    free(c);
    free(pr);
    free(pc);
    return rel <= 1e-10 ? 0 : 1;
  }
}

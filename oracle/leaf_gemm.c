/*
 * leaf_gemm.c -- TEST INFRASTRUCTURE ONLY.  The per-leaf product the
 * reference delegates to np.matmul / OpenBLAS (multiply.py:255).  OpenBLAS's
 * internal FMA/blocking order is not part of the reference (it is a
 * third-party dependency, pinned only as numpy>=1.24, pyproject.toml:10), so
 * C is compared by tolerance (1e-13 relative Frobenius vs the reference's
 * own C in tests/golden), never bit-for-bit.  Compiled with FMA contraction
 * allowed and AVX2 vectorisation, row-axpy (i-t-j) loop order.
 */
#include <stdint.h>
#include <string.h>

void oracle_leaf_gemm_f64(const double *a, const double *b, int64_t lda, int32_t leaf, double *p) {
  memset(p, 0, sizeof(double) * leaf * leaf);
  for (int r = 0; r < leaf; ++r) {
    double *pr = p + (int64_t)r * leaf;
    for (int t = 0; t < leaf; ++t) {
      const double av = a[(int64_t)r * lda + t];
      const double *bt = b + (int64_t)t * lda;
      for (int c = 0; c < leaf; ++c) pr[c] += av * bt[c];
    }
  }
}

void oracle_leaf_gemm_f32(const float *a, const float *b, int64_t lda, int32_t leaf, float *p) {
  memset(p, 0, sizeof(float) * leaf * leaf);
  for (int r = 0; r < leaf; ++r) {
    float *pr = p + (int64_t)r * leaf;
    for (int t = 0; t < leaf; ++t) {
      const float av = a[(int64_t)r * lda + t];
      const float *bt = b + (int64_t)t * lda;
      for (int c = 0; c < leaf; ++c) pr[c] += av * bt[c];
    }
  }
}

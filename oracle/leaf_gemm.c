/*
 * leaf_gemm.c -- TEST INFRASTRUCTURE ONLY.  The per-leaf product the
 * reference delegates to np.matmul / OpenBLAS (multiply.py:255).  OpenBLAS's
 * internal FMA/blocking order is not part of the reference (a third-party
 * dependency, pinned only as numpy>=1.24, pyproject.toml:10).  For these leaf
 * sizes the build container's OpenBLAS 0.3.30 (SkylakeX kernels) accumulates
 * each output element as one sequential FMA chain over the inner index from
 * zero; this row-axpy (i-t-j) loop, compiled with FMA contraction, forms the
 * same chain, so C matches the reference's own C in tests/golden bit for bit
 * (tests/test_oracle.py).  A different BLAS build could order its FMAs
 * differently -- the contract bar is 1e-12 relative Frobenius.
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

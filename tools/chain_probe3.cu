// K1 chain inner-loop variants: cycles per element of one sequential
// acc = rn(acc + rn(x*x)) chain per lane, data staged in shared memory.
//  mode 0: pre-squared values, LDS.128 x8 then 16 DADD            (current K1 chain warp)
//  mode 1: raw values, LDS.128 x8 then 16 x (DMUL, DADD)           (chain warp squares)
//  mode 2: mode 1 with the next batch's LDS issued before this batch's math
//  mode 3: registers only, DADD chain                              (floor)
//  mode 4: registers only, DMUL + DADD chain
#include <cstdio>
#include <cuda_runtime.h>
constexpr int STRIDE = 528;  // bytes per lane row (512 + 16 pad)
__device__ double g_src[1 << 22];
__global__ void chain(double *out, long long *cyc, int reps, int mode) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *base = sm + warp * 32 * STRIDE;
  for (int i = lane; i < 32 * STRIDE / 8; i += 32)
    ((double *)base)[i] = mode == 8 ? 1e-310 * (1 + i % 7) : mode == 9 ? 1e-200 * (1 + i % 7) : 1.0 + i * 1e-7;
  __syncwarp();
  const unsigned char *pp = base + lane * STRIDE;
  double acc = 0.0;
  long long t0 = clock64();
  if (mode == 11 && warp > 0) {
    unsigned char *dst = base;
    for (int c = 0; c < reps * 8; ++c) {
      for (int q = 0; q < 16; ++q) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + (q * 32 + lane) * 16 % (32 * STRIDE - 16));
        const double *g = g_src + ((size_t)(blockIdx.x * 8 + warp) * 4096 + c * 512 + q * 32 + lane) * 2 % ((1 << 22) - 2);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
      }
      asm volatile("cp.async.commit_group;\n");
      asm volatile("cp.async.wait_group 4;\n");
    }
    asm volatile("cp.async.wait_group 0;\n");
    return;
  }
  if (mode >= 5 && mode <= 7 && warp > 0) {
    // background FP64 load on the other warps: mode 5 DMUL stream, mode 6 DADD stream,
    // mode 7 integer stream
    double r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) r[u] = 1.0 + (lane + u) * 1e-9;
    unsigned ir[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) ir[u] = lane + u;
    for (int c = 0; c < reps * 16; ++c) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (mode == 5) r[u] = __dmul_rn(r[u], 1.0000001);
        else if (mode == 6) r[u] = __dadd_rn(r[u], 1e-9);
        else ir[u] = ir[u] * 1664525u + 1013904223u;
      }
    }
    double z = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) z += r[u] + ir[u];
    out[threadIdx.x + blockIdx.x * blockDim.x] = z;
    return;
  }
  const bool active8 = mode == 10;
  if (mode == 12 || mode == 13) {
    long long t0b = clock64();
    for (int c = 0; c < reps; ++c) {
      double2 w[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) w[u] = *reinterpret_cast<const double2 *>(pp + 16 * u);
      __syncwarp();
      if (mode == 12) {
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          acc = __dadd_rn(acc, w[u].x);
          acc = __dadd_rn(acc, w[u].y);
        }
      } else {  // two interleaved half-chains combined at the end (NOT the reference order; timing only)
        double a2 = 0.0;
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          acc = __dadd_rn(acc, w[u].x);
          a2 = __dadd_rn(a2, w[u].y);
        }
        acc += a2;
      }
    }
    long long t1b = clock64();
    out[threadIdx.x + blockIdx.x * blockDim.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1b - t0b;
    return;
  }
  if (mode >= 5) mode = 0;
  __syncwarp();
  if (active8 && lane >= 8) { out[threadIdx.x + blockIdx.x * blockDim.x] = 0; return; }
  if (mode == 0 || mode == 1) {
    for (int c = 0; c < reps; ++c) {
      for (int v = 0; v < 32; v += 8) {
        double2 w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = *reinterpret_cast<const double2 *>(pp + 16 * (v + u));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (mode == 0) {
            acc = __dadd_rn(acc, w[u].x);
            acc = __dadd_rn(acc, w[u].y);
          } else {
            acc = __dadd_rn(acc, __dmul_rn(w[u].x, w[u].x));
            acc = __dadd_rn(acc, __dmul_rn(w[u].y, w[u].y));
          }
        }
      }
    }
  } else if (mode == 2) {
    double2 w[8], nx[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) w[u] = *reinterpret_cast<const double2 *>(pp + 16 * u);
    for (int c = 0; c < reps; ++c) {
      for (int v = 0; v < 32; v += 8) {
        const int vn = (v + 8) & 31;
#pragma unroll
        for (int u = 0; u < 8; ++u) nx[u] = *reinterpret_cast<const double2 *>(pp + 16 * (vn + u));
        double sq[16];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          sq[2 * u] = __dmul_rn(w[u].x, w[u].x);
          sq[2 * u + 1] = __dmul_rn(w[u].y, w[u].y);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, sq[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = nx[u];
      }
    }
  } else {
    double r[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) r[u] = 1.0 + (lane + u) * 1e-9;
    for (int c = 0; c < reps * 4; ++c) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (mode == 3) acc = __dadd_rn(acc, r[u]);
        else acc = __dadd_rn(acc, __dmul_rn(r[u], r[u]));
      }
      r[c & 15] += 1e-12;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double *o;
  long long *c;
  cudaMalloc(&o, 8 * 4096 * 64);
  cudaMallocManaged(&c, 8);
  const int reps = 64;  // x 64 elements per lane
  for (int warps : {6, 8}) {
    for (int mode = 0; mode < 14; ++mode) {
      const int smem = warps * 32 * STRIDE;
      cudaFuncSetAttribute(chain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      chain<<<148, 32 * warps, smem>>>(o, c, reps, mode);
      cudaDeviceSynchronize();
      chain<<<148, 32 * warps, smem>>>(o, c, reps, mode);
      cudaDeviceSynchronize();
      printf("warps/SM %2d mode %d: %.2f cycles/element (%s)\n", warps, mode,
             (double)*c / (reps * 64), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
// (see mode 11: cp.async streaming helper warps; appended variant below)

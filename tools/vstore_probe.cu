// Dev probe: HBM write rate of the input transform's V store pattern
// V[xi][c][t] (t contiguous) for c4's geometry, as a function of the t-run
// length each CTA writes per (xi, c): run = 49 tiles (one depth tile, the
// current slab), 98 (two), 196 (two samples).  Values are constants: this
// isolates the store side.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k(float* V, int run, int P, int C, long long T_s, int nslab_per_c) {
  const int w = blockIdx.x;
  const int c = w / nslab_per_c;
  const long long t0 = (long long)(w % nslab_per_c) * run;
  const long long pstride = (long long)C * T_s;
  float* vb = V + (long long)c * T_s + t0;
  for (int i = threadIdx.x; i < P * run; i += blockDim.x) {
    const int xi = i / run, tl = i - xi * run;
    vb[xi * pstride + tl] = (float)i;
  }
}

// the real kernel's order: one work item per (xi0, tile) writes alpha^2 values
__global__ void __launch_bounds__(256) k2(float* V, int run, int P, int C, long long T_s, int nslab_per_c) {
  const int w = blockIdx.x;
  const int c = w / nslab_per_c;
  const long long t0 = (long long)(w % nslab_per_c) * run;
  const long long pstride = (long long)C * T_s;
  float* vb = V + (long long)c * T_s + t0;
  const int A2 = 36, A = 6;
  for (int it = threadIdx.x; it < A * run; it += blockDim.x) {
    const int xi0 = it / run, tl = it - xi0 * run;
    float* vo = vb + tl + (long long)xi0 * A2 * pstride;
#pragma unroll
    for (int j = 0; j < A2; ++j) vo[j * pstride] = (float)j;
  }
}

// k2's pattern over `nsub` consecutive 49-tile slabs of the same c, one after
// the other (a CTA looping over slabs)
__global__ void __launch_bounds__(256) k3(float* V, int nsub, int P, int C, long long T_s, int nslab_per_c) {
  const int run = 49;
  const int w = blockIdx.x;
  const int c = w / nslab_per_c;
  const long long pstride = (long long)C * T_s;
  const int A2 = 36, A = 6;
  for (int sub = 0; sub < nsub; ++sub) {
    const long long t0 = ((long long)(w % nslab_per_c) * nsub + sub) * run;
    float* vb = V + (long long)c * T_s + t0;
    for (int it = threadIdx.x; it < A * run; it += blockDim.x) {
      const int xi0 = it / run, tl = it - xi0 * run;
      float* vo = vb + tl + (long long)xi0 * A2 * pstride;
#pragma unroll
      for (int j = 0; j < A2; ++j) vo[j * pstride] = (float)j;
    }
    __syncthreads();
  }
}

// k2's pattern with lanes padded to whole warps per xi0 (64 lanes per 49-tile
// run: no warp straddles two xi0 runs)
__global__ void __launch_bounds__(384) k4(float* V, int run, int P, int C, long long T_s, int nslab_per_c) {
  const int w = blockIdx.x;
  const int c = w / nslab_per_c;
  const long long t0 = (long long)(w % nslab_per_c) * run;
  const long long pstride = (long long)C * T_s;
  float* vb = V + (long long)c * T_s + t0;
  const int A2 = 36, A = 6;
  const int rp = (run + 31) / 32 * 32;
  for (int it = threadIdx.x; it < A * rp; it += blockDim.x) {
    const int xi0 = it / rp, tl = it - xi0 * rp;
    if (tl >= run) continue;
    float* vo = vb + tl + (long long)xi0 * A2 * pstride;
#pragma unroll
    for (int j = 0; j < A2; ++j) vo[j * pstride] = (float)j;
  }
}

// k2 with a per-slab t stride `pitch` >= run (pitch = run: packed, current
// layout; pitch = run rounded up to 8 floats: 32-byte aligned runs)
__global__ void __launch_bounds__(256) k5(float* V, int run, int pitch, int P, int C, long long T_s, int nslab_per_c) {
  const int w = blockIdx.x;
  const int c = w / nslab_per_c;
  const long long t0 = (long long)(w % nslab_per_c) * pitch;
  const long long pstride = (long long)C * T_s;
  float* vb = V + (long long)c * T_s + t0;
  const int A2 = 36, A = 6;
  for (int it = threadIdx.x; it < A * run; it += blockDim.x) {
    const int xi0 = it / run, tl = it - xi0 * run;
    float* vo = vb + tl + (long long)xi0 * A2 * pstride;
#pragma unroll
    for (int j = 0; j < A2; ++j) vo[j * pstride] = (float)j;
  }
}

int main() {
  const int P = 216, C = 256, B = 32, Tps = 98;
  const long long T = (long long)B * Tps, T_s = (T + 127) / 128 * 128;
  float* V;
  cudaMalloc(&V, (size_t)P * C * T_s * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int kern = 0; kern < 2; ++kern)
    for (int run : {49, 98, 196, 392}) {
      const int nslab_per_c = (int)(T / run);
      const int grid = nslab_per_c * C;
      for (int w = 0; w < 2; ++w)
        kern ? k2<<<grid, 256>>>(V, run, P, C, T_s, nslab_per_c) : k<<<grid, 256>>>(V, run, P, C, T_s, nslab_per_c);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r)
        kern ? k2<<<grid, 256>>>(V, run, P, C, T_s, nslab_per_c) : k<<<grid, 256>>>(V, run, P, C, T_s, nslab_per_c);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      const double bytes = (double)P * C * T * 4;
      printf("kern %d run %3d: %.1f us  %.0f GB/s  %s\n", kern, run, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  for (int nsub : {1, 2, 4, 8}) {
    const int nslab_per_c = (int)(T / (49 * nsub));
    const int grid = nslab_per_c * C;
    for (int w = 0; w < 2; ++w) k3<<<grid, 256>>>(V, nsub, P, C, T_s, nslab_per_c);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k3<<<grid, 256>>>(V, nsub, P, C, T_s, nslab_per_c);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("k3 nsub %d (CTA loops over 49-tile slabs): %.1f us  %.0f GB/s\n", nsub, ms * 1e3,
           (double)P * C * T * 4 / (ms * 1e-3) / 1e9);
  }
  for (int pitch : {98, 104, 128}) {
    const int run = 98;
    const long long Tp = (long long)B * pitch, T_sp = (Tp + 127) / 128 * 128;
    float* V2;
    cudaMalloc(&V2, (size_t)P * C * T_sp * 4);
    const int nslab_per_c = B;
    const int grid = nslab_per_c * C;
    for (int w = 0; w < 2; ++w) k5<<<grid, 256>>>(V2, run, pitch, P, C, T_sp, nslab_per_c);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k5<<<grid, 256>>>(V2, run, pitch, P, C, T_sp, nslab_per_c);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("k5 run 98 pitch %d: %.1f us  %.0f GB/s of V\n", pitch, ms * 1e3, (double)P * C * T * 4 / (ms * 1e-3) / 1e9);
    cudaFree(V2);
  }
  for (int run : {49, 98}) {
    const int nslab_per_c = (int)(T / run);
    const int grid = nslab_per_c * C;
    for (int w = 0; w < 2; ++w) k4<<<grid, 384>>>(V, run, P, C, T_s, nslab_per_c);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k4<<<grid, 384>>>(V, run, P, C, T_s, nslab_per_c);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("k4 run %d (warp-aligned xi0 runs): %.1f us  %.0f GB/s\n", run, ms * 1e3,
           (double)P * C * T * 4 / (ms * 1e-3) / 1e9);
  }
  return 0;
}

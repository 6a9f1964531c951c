// FP64 pipe microbenchmarks for B200 (sm_100a): DMMA (mma.sync .f64) and DFMA peaks,
// whether they share the FP64 datapath, and DMMA's rounding behaviour.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_fp64.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void k_dmma(double* out, int iters, double seed) {
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dfma(double* out, int iters, double seed) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = i;
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// mixed: per iteration NACC DMMA + NF DFMA per thread
template <int NACC, int NF>
__global__ void k_mixed(double* out, int iters, double seed) {
  double acc[NACC][2];
  double f[NF];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
#pragma unroll
  for (int i = 0; i < NF; ++i) f[i] = i;
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9, c = 1.0 - 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i][0], acc[i][1], a, b);
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = fma(f[i], c, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += f[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// Rounding behaviour: one warp, D = A(8x4) * B(4x8) + C, compare with sequential fma in k order.
__global__ void k_dmma_round(const double* A, const double* B, const double* C, double* D) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a = A[g * 4 + t];      // A row-major 8x4
  double b = B[t * 8 + g];      // B 4x8 row-major: B[k][n]
  double d0 = C[g * 8 + 2 * t], d1 = C[g * 8 + 2 * t + 1];
  dmma(d0, d1, a, b);
  D[g * 8 + 2 * t] = d0; D[g * 8 + 2 * t + 1] = d1;
}

static double now_ms(cudaEvent_t a, cudaEvent_t b) { float ms; cudaEventElapsedTime(&ms, a, b); return ms; }

// `mb peaks`: the two roofline denominators bench.py uses, as one JSON line — DMMA burst (best of
// 10 single launches of ~10 ms) and sustained (back to back for ~4 s), the kernel and shape of the
// sweep's best row (2 CTAs x 256 threads per SM, 8 independent accumulators). tools/fp64_peaks.py
// runs it under an nvidia-smi sampler and writes profiles/fp64_peaks.json.
static int peaks_main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = p.multiProcessorCount * 2, thr = 256, iters = 40000;
  const double flops = (double)grid * (thr / 32) * iters * 8 * 512.0;
  k_dmma<8><<<grid, thr>>>(out, 100, 1.0); CK(cudaDeviceSynchronize());
  double best = 1e30;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_dmma<8><<<grid, thr>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    const double ms = now_ms(e0, e1);
    if (ms < best) best = ms;
  }
  int reps = 0;
  cudaEventRecord(e0);
  double ms = 0;
  while (ms < 4000.0) {
    for (int i = 0; i < 40; ++i, ++reps) k_dmma<8><<<grid, thr>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    ms = now_ms(e0, e1);
  }
  printf("{\"dmma_tflops_burst\": %.4f, \"dmma_tflops_sustained\": %.4f, \"burst_ms\": %.4f, "
         "\"sustained_ms\": %.1f, \"sustained_launches\": %d, \"grid\": %d, \"threads\": %d, "
         "\"kernel\": \"mma.sync.m8n8k4.f64 (DMMA.8x8x4), 8 accumulators per warp\"}\n",
         flops / best / 1e9, flops * reps / ms / 1e9, best, ms, reps, grid, thr);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 'p') return peaks_main();
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d L2 %d B smem/SM %zu clock(kHz) %d\n", p.name, p.multiProcessorCount, p.l2CacheSize,
         p.sharedMemPerMultiprocessor, clk);
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // DMMA peak sweep
  for (int bpsm : {1, 2, 4}) for (int thr : {128, 256}) {
    int grid = sms * bpsm, iters = 20000;
    k_dmma<8><<<grid, thr>>>(out, 100, 1.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_dmma<8><<<grid, thr>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    double ms = now_ms(e0, e1);
    double flops = (double)grid * (thr / 32) * iters * 8 * 512.0;
    printf("DMMA nacc=8 grid=%d thr=%d: %.3f ms  %.2f TFLOP/s\n", grid, thr, ms, flops / ms / 1e9);
  }
  // DMMA sustained (~4 s)
  {
    int grid = sms * 2, thr = 256, iters = 20000;
    double flops1 = (double)grid * (thr / 32) * iters * 8 * 512.0;
    cudaEventRecord(e0);
    int reps = 0;
    for (; reps < 400; ++reps) k_dmma<8><<<grid, thr>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    double ms = now_ms(e0, e1);
    printf("DMMA sustained %d launches %.1f ms: %.2f TFLOP/s\n", reps, ms, flops1 * reps / ms / 1e9);
  }
  for (int bpsm : {2, 4}) for (int thr : {256}) {
    int grid = sms * bpsm, iters = 20000;
    k_dfma<8><<<grid, thr>>>(out, 100, 1.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_dfma<8><<<grid, thr>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    double ms = now_ms(e0, e1);
    double flops = (double)grid * thr * iters * 8 * 2.0;
    printf("DFMA grid=%d thr=%d: %.3f ms  %.2f TFLOP/s\n", grid, thr, ms, flops / ms / 1e9);
  }
  {
    int grid = sms * 2, thr = 256, iters = 20000;
    k_mixed<8, 8><<<grid, thr>>>(out, 100, 1.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_mixed<8, 8><<<grid, thr>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    double ms = now_ms(e0, e1);
    double fm = (double)grid * (thr / 32) * iters * 8 * 512.0;
    double ff = (double)grid * thr * iters * 8 * 2.0;
    printf("MIXED 8 DMMA + 8 DFMA per thread-iter: %.3f ms; DMMA part %.2f TF, DFMA part %.2f TF, sum %.2f\n",
           ms, fm / ms / 1e9, ff / ms / 1e9, (fm + ff) / ms / 1e9);
    k_mixed<8, 2><<<grid, thr>>>(out, 100, 1.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_mixed<8, 2><<<grid, thr>>>(out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    ms = now_ms(e0, e1);
    ff = (double)grid * thr * iters * 2 * 2.0;
    printf("MIXED 8 DMMA + 2 DFMA per thread-iter: %.3f ms; DMMA part %.2f TF, DFMA part %.2f TF\n",
           ms, fm / ms / 1e9, ff / ms / 1e9);
  }
  // Rounding test
  {
    const int T = 2000;
    int seq_mis = 0, exact_mis = 0, pair_mis = 0;
    double *dA, *dB, *dC, *dD; CK(cudaMalloc(&dA, 32 * 8)); CK(cudaMalloc(&dB, 32 * 8));
    CK(cudaMalloc(&dC, 64 * 8)); CK(cudaMalloc(&dD, 64 * 8));
    srand(1);
    for (int trial = 0; trial < T; ++trial) {
      double A[32], B[32], C[64], D[64];
      auto rnd = []() { return ((double)rand() / RAND_MAX - 0.5) * pow(2.0, (rand() % 40) - 20); };
      for (int i = 0; i < 32; ++i) { A[i] = rnd(); B[i] = rnd(); }
      for (int i = 0; i < 64; ++i) C[i] = rnd();
      cudaMemcpy(dA, A, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, B, 256, cudaMemcpyHostToDevice);
      cudaMemcpy(dC, C, 512, cudaMemcpyHostToDevice);
      k_dmma_round<<<1, 32>>>(dA, dB, dC, dD);
      cudaMemcpy(D, dD, 512, cudaMemcpyDeviceToHost);
      for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) {
        double s = C[r * 8 + c];
        for (int kk = 0; kk < 4; ++kk) s = fma(A[r * 4 + kk], B[kk * 8 + c], s);
        if (s != D[r * 8 + c]) seq_mis++;
        long double e = C[r * 8 + c];
        for (int kk = 0; kk < 4; ++kk) e += (long double)A[r * 4 + kk] * (long double)B[kk * 8 + c];
        if ((double)e != D[r * 8 + c]) exact_mis++;
        double s2 = C[r * 8 + c];
        for (int kk = 3; kk >= 0; --kk) s2 = fma(A[r * 4 + kk], B[kk * 8 + c], s2);
        if (s2 != D[r * 8 + c]) pair_mis++;
      }
    }
    printf("DMMA rounding over %d elems: seq-fma(k asc) mismatches %d, seq-fma(k desc) %d, x87-exact-ish %d\n",
           T * 64, seq_mis, pair_mis, exact_mis);
  }
  return 0;
}

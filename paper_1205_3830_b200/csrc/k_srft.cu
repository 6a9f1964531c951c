// k_srft.cu — the paper's own randomisation Y = S F D A (§2, Eqs. 4–7; NEXT-1 of
// SURVEY.md §8(f)), on B200: an FFT factorisation whose heavy half runs on the DMMA pipe.
//
// With m = m1 * R (R = 16) and i = i1 + m1 * i2, the sampled DFT rows factor as
//     Y(k, c) = sum_{i1} W_m^{(s_k i1) mod m} * Z_c(i1, s_k mod R),
//     Z_c(i1, r) = sum_{i2 < R} W_R^{r i2} * d(i1 + m1 i2) * A(i1 + m1 i2, c)
// (W_N = e^{-2 pi i / N}; W_m^{s m1 i2} = W_R^{s i2}). So:
//   pass 1 (k_srft_pass1): D-scaling and the R-point DFT along i2, one thread per (i1, c), radix-4
//     x radix-4 in registers, coalesced along i1 — one read of A, one write of Z (HBM-bound);
//   pass 2: for each residue r, the rows k with s_k mod R = r form one small complex GEMM
//     Y_r (l_r x n) = W_r (l_r x m1) . Z^(r) (m1 x n) on the same complex-product kernel as the
//     Gaussian sketch (k_zgemm3m.cu, Gauss's three products; the ordered k_zgemm.cu with
//     RID_SKETCH_4M=1) — 6 (or 8) l m n / R real flops instead of the dense 8 l m n.
// Plan (docs/RNG.md §7): d_i = (cos, sin)(2 pi u1) of Philox (i, 0, s_phase, 0) via the spec'd
// sincos, s_k = x0 & (m - 1) of Philox (k, 0, s_sample, 0); W entries from the same sincos on
// u = ((s_k i1) mod m) / m. Agreement with the oracle's direct ascending sum is to rounding.
#include <cstdlib>

#include "rid_device.cuh"
#include "rid_internal.h"

namespace rid {

constexpr int kSrftR = 16;

__global__ void k_srft_plan(uint64_t seed, uint32_t s_phase, uint32_t s_sample, int64_t m,
                            int64_t l, double2* __restrict__ d, int64_t* __restrict__ samples) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 x = philox4x32_10(make_uint4((uint32_t)i, 0u, s_phase, 0u), k0, k1);
    d[i] = rid_cossin2pi(u01_from(x.x, x.y));
    if (i < l) {
      const uint4 y = philox4x32_10(make_uint4((uint32_t)i, 0u, s_sample, 0u), k0, k1);
      samples[i] = (int64_t)(y.x & (uint32_t)(m - 1));
    }
  }
  // l may exceed m (sampling with replacement)
  for (int64_t i = m + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < l;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 y = philox4x32_10(make_uint4((uint32_t)i, 0u, s_sample, 0u), k0, k1);
    samples[i] = (int64_t)(y.x & (uint32_t)(m - 1));
  }
}

// Stable counting sort of the samples by residue s mod R (one CTA): order[pos] = k, offs[r].
__global__ void k_srft_group(const int64_t* __restrict__ samples, int64_t l, int* __restrict__ order,
                             int* __restrict__ offs) {
  __shared__ int cnt[kSrftR + 1];
  if (threadIdx.x <= kSrftR) cnt[threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t k = 0; k < l; ++k) cnt[(int)(samples[k] % kSrftR) + 1]++;
    for (int r = 0; r < kSrftR; ++r) cnt[r + 1] += cnt[r];
    for (int r = 0; r <= kSrftR; ++r) offs[r] = cnt[r];
    for (int64_t k = 0; k < l; ++k) order[cnt[(int)(samples[k] % kSrftR)]++] = (int)k;
  }
}

// Wg(k', i1) = W_m^{(s_{order[k']} i1) mod m}, column-major l x m1 (ld = l)
__global__ void k_srft_wgen(const int64_t* __restrict__ samples, const int* __restrict__ order,
                            int64_t l, int64_t m, int64_t m1, double2* __restrict__ Wg) {
  const int64_t total = l * m1;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kk = q % l, i1 = q / l;
    const uint64_t t = ((uint64_t)samples[order[kk]] * (uint64_t)i1) & (uint64_t)(m - 1);
    const double2 cs = rid_cossin2pi(__ddiv_rn((double)t, (double)m));  // exact: m = 2^p
    Wg[q] = make_double2(cs.x, -cs.y);
  }
}

// Ws(prow(k'), i1) = Re Wg(k', i1) + Im Wg(k', i1) with each residue group starting on an even
// row (ps[r] = sum of the earlier groups' sizes rounded up to even; pad rows zero): the 3M
// kernel's non-swizzled TMA boxes of the plane must start on a 16-byte boundary.
__global__ void k_srft_wsum(const double2* __restrict__ Wg, int64_t l, int64_t m1,
                            const int* __restrict__ offs, double* __restrict__ Ws, int64_t ldws) {
  __shared__ int so[kSrftR + 1], sp[kSrftR + 1];
  if (threadIdx.x == 0) {
    sp[0] = 0;
    for (int r = 0; r <= kSrftR; ++r) so[r] = offs[r];
    for (int r = 0; r < kSrftR; ++r) sp[r + 1] = sp[r] + ((so[r + 1] - so[r] + 1) & ~1);
  }
  __syncthreads();
  const int64_t total = ldws * m1;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i1 = q / ldws, pr = q % ldws;
    int r = 0;
    while (r < kSrftR - 1 && pr >= sp[r + 1]) ++r;
    const int64_t kk = so[r] + (pr - sp[r]);
    double v = 0.0;
    if (pr < sp[kSrftR] && kk < so[r + 1]) {
      const double2 w = Wg[i1 * l + kk];
      v = __dadd_rn(w.x, w.y);
    }
    Ws[q] = v;
  }
}

// complex helpers
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // * (-i)

// 4-point DFT (forward): X_q = sum_p x_p W_4^{pq}
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 a = cadd(x0, x2), b = csub(x0, x2), c = cadd(x1, x3), e = mul_mi(csub(x1, x3));
  x0 = cadd(a, c);
  x2 = csub(a, c);
  x1 = cadd(b, e);
  x3 = csub(b, e);
}

__global__ void __launch_bounds__(128) k_srft_pass1(const double2* __restrict__ A, int64_t lda,
                                                    int64_t m1, int64_t n_loc,
                                                    const double2* __restrict__ d,
                                                    double2* __restrict__ Z) {
  // W_16^e, e = 0..9 (the twiddles of the 4 x 4 split: W_16^{p q}, p, q < 4)
  const double c1 = 0.92387953251128674, s1 = 0.38268343236508978, h = 0.70710678118654757;
  const double2 W[10] = {make_double2(1, 0),   make_double2(c1, -s1), make_double2(h, -h),
                         make_double2(s1, -c1), make_double2(0, -1),  make_double2(-s1, -c1),
                         make_double2(-h, -h),  make_double2(-c1, -s1), make_double2(-1, 0),
                         make_double2(-c1, s1)};
  const int64_t i1 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (i1 >= m1) return;
  const double2* a = A + c * lda + i1;
  double2 x[16];
#pragma unroll
  for (int i2 = 0; i2 < 16; ++i2) x[i2] = cmul(__ldg(d + i1 + m1 * i2), __ldcs(a + m1 * i2));
  // 16 = 4 x 4, i2 = p + 4 q: first DFT-4 over q (stride 4) for each p, twiddle W_16^{p r1},
  // then DFT-4 over p; output index r = r1 + 4 r2.
#pragma unroll
  for (int p = 0; p < 4; ++p) dft4(x[p], x[p + 4], x[p + 8], x[p + 12]);  // x[p + 4 r1]
#pragma unroll
  for (int p = 1; p < 4; ++p)
#pragma unroll
    for (int r1 = 1; r1 < 4; ++r1) x[p + 4 * r1] = cmul(x[p + 4 * r1], W[p * r1]);
#pragma unroll
  for (int r1 = 0; r1 < 4; ++r1) dft4(x[4 * r1], x[4 * r1 + 1], x[4 * r1 + 2], x[4 * r1 + 3]);
  // x[4 r1 + r2] now holds output r = r1 + 4 r2
#pragma unroll
  for (int r1 = 0; r1 < 4; ++r1)
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2) {
      const int r = r1 + 4 * r2;
      Z[((int64_t)r * n_loc + c) * m1 + i1] = x[4 * r1 + r2];
    }
}

__global__ void k_srft_scatter(const double2* __restrict__ Yg, const int* __restrict__ order,
                               int64_t l, int64_t n_loc, double2* __restrict__ Y, int64_t ldy) {
  const int64_t total = l * n_loc;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kk = q % l, c = q / l;
    Y[c * ldy + order[kk]] = Yg[q];
  }
}

// Column chunk of the two passes: Z is as large as A's chunk, so a chunk of ~4 GiB of A bounds
// the workspace (C5: 2048 columns per chunk) while every GEMM still has >= 2 CTAs per SM.
int64_t srft_chunk_cols(int64_t m, int64_t n_loc) {
  int64_t c = ((int64_t)4 << 30) / (16 * m);
  if (c < 64) c = 64;
  return c < n_loc ? c : n_loc;
}

size_t srft_work_bytes(int64_t m, int64_t l, int64_t n_loc) {
  const int64_t m1 = m / kSrftR, ch = srft_chunk_cols(m, n_loc);
  return sizeof(double2) * ((size_t)m + (size_t)l * m1 + (size_t)kSrftR * m1 * ch +
                            (size_t)l * ch) +
         sizeof(double) * (size_t)(rsum_ld(l) + kSrftR) * m1 +  // Re Wg + Im Wg, padded
         sizeof(int64_t) * (size_t)l + sizeof(int) * ((size_t)l + kSrftR + 1) + 2304;
}

cudaError_t srft_sketch(uint64_t seed, bool retry, int64_t l, const double2* A, int64_t m,
                        int64_t n, int64_t n_loc, int64_t lda, double2* Y, int64_t ldy, void* work,
                        double2* splitk, size_t splitk_elems, int num_sms, cudaStream_t st,
                        int* launches) {
  if (m < kSrftR || (m & (m - 1)) != 0) return cudaErrorInvalidValue;
  const int64_t m1 = m / kSrftR, ch = srft_chunk_cols(m, n_loc);
  if (ch > 65535) return cudaErrorInvalidConfiguration;
  char* w = (char*)work;
  auto take = [&](size_t bytes) {
    char* p = w;
    w += (bytes + 255) & ~(size_t)255;
    return (void*)p;
  };
  double2* d = (double2*)take(sizeof(double2) * m);
  double2* Wg = (double2*)take(sizeof(double2) * l * m1);
  const int64_t ldws = rsum_ld(l) + kSrftR;  // >= every padded group layout, even
  double* Wgs = (double*)take(sizeof(double) * ldws * m1);  // Re Wg + Im Wg (3M sums)
  double2* Z = (double2*)take(sizeof(double2) * kSrftR * m1 * ch);
  double2* Yg = (double2*)take(sizeof(double2) * l * ch);
  int64_t* samples = (int64_t*)take(sizeof(int64_t) * l);
  int* order = (int*)take(sizeof(int) * l);
  int* offs = (int*)take(sizeof(int) * (kSrftR + 1));
  const uint32_t sp = retry ? 22u : 6u, ss = retry ? 23u : 7u;
  int64_t blocks = ((m > l ? m : l) + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_srft_plan<<<(unsigned)blocks, 256, 0, st>>>(seed, sp, ss, m, l, d, samples);
  k_srft_group<<<1, 32, 0, st>>>(samples, l, order, offs);
  int64_t wb = (l * m1 + 255) / 256;
  if (wb > 8192) wb = 8192;
  k_srft_wgen<<<(unsigned)wb, 256, 0, st>>>(samples, order, l, m, m1, Wg);
  {
    int64_t sb = (ldws * m1 + 255) / 256;
    if (sb > 8192) sb = 8192;
    k_srft_wsum<<<(unsigned)sb, 256, 0, st>>>(Wg, l, m1, offs, Wgs, ldws);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int hoffs[kSrftR + 1];
  e = cudaMemcpyAsync(hoffs, offs, sizeof(hoffs), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  *launches += 4;
  for (int64_t c0 = 0; c0 < n_loc; c0 += ch) {
    const int64_t nc = (c0 + ch <= n_loc) ? ch : n_loc - c0;
    dim3 g1((unsigned)((m1 + 127) / 128), (unsigned)nc);
    k_srft_pass1<<<g1, 128, 0, st>>>(A + c0 * lda, lda, m1, nc, d, Z);
    *launches += 1;
    if (sketch_mults() == 3) {  // the 16 residue products in one batched launch (no K split)
      Z3Batch bt{};
      for (int r = 0; r < kSrftR; ++r) {
        const int64_t lr = hoffs[r + 1] - hoffs[r];
        if (lr == 0) continue;
        bt.roff[bt.n] = hoffs[r];
        bt.boff[bt.n] = (int64_t)r * m1 * nc;
        bt.coff[bt.n] = hoffs[r];
        bt.mout[bt.n] = lr;
        ++bt.n;
      }
      const char* v = select_env("RID_Z3_TMA");
      if (v && atoi(v) == 0) {
        e = zgemm3m_batched(Wg, l, Z, m1, Yg, l, bt, nc, m1, st);
        if (e != cudaSuccess) return e;
        *launches += 1;
      } else {
        // each residue's l_r rows cut into 48-, 40- and 24-row tiles with the fewest padded rows
        // (l_r ~ l/16 ± 25%: one fixed height pads 20-30% of the residue products), one batched
        // launch per tile height
        Z3Batch bh[3] = {};
        const int hts[3] = {48, 40, 24};
        int64_t ps[kSrftR + 1];  // even-padded group starts in Wgs (k_srft_wsum)
        ps[0] = 0;
        for (int r = 0; r < kSrftR; ++r) ps[r + 1] = ps[r] + ((hoffs[r + 1] - hoffs[r] + 1) & ~1);
        int zr[kZ3BatchMax];  // residue of item z of bt
        for (int r = 0, z = 0; r < kSrftR; ++r)
          if (hoffs[r + 1] > hoffs[r]) zr[z++] = r;
        for (int z = 0; z < bt.n; ++z) {
          const int64_t lr = bt.mout[z];
          int64_t best = INT64_MAX;
          int cnt[3] = {0, 0, 0};
          for (int a3 = 0; a3 <= (int)((lr + 47) / 48); ++a3)
            for (int b3 = 0; b3 <= 2; ++b3)
              for (int c3 = 0; c3 <= 2; ++c3) {
                const int64_t cover = 48 * a3 + 40 * b3 + 24 * c3;
                if (cover < lr) continue;
                const int64_t cost = (cover - lr) * 16 + a3 + b3 + c3;  // padding, then tiles
                if (cost < best) {
                  best = cost;
                  cnt[0] = a3;
                  cnt[1] = b3;
                  cnt[2] = c3;
                }
              }
          int64_t row = 0;
          for (int h = 0; h < 3 && row < lr; ++h) {
            if (cnt[h] == 0) continue;
            const int64_t rows = (lr - row < (int64_t)cnt[h] * hts[h]) ? lr - row : (int64_t)cnt[h] * hts[h];
            Z3Batch& q = bh[h];
            q.roff[q.n] = bt.roff[z] + row;
            q.soff[q.n] = ps[zr[z]] + row;  // row is a multiple of 48 / 40 / 24: even
            q.boff[q.n] = bt.boff[z];
            q.coff[q.n] = bt.coff[z] + row;
            q.mout[q.n] = rows;
            ++q.n;
            row += rows;
          }
        }
        for (int h = 0; h < 3; ++h) {
          if (bh[h].n == 0) continue;
          e = zgemm3m_tma_batched_h(Wg, l, l, Z, m1, kSrftR * nc, Yg, l, bh[h], nc, m1, hts[h], st,
                                    Wgs, ldws, ps[kSrftR]);
          if (e != cudaSuccess) return e;
          *launches += 1;
        }
      }
    } else {
      for (int r = 0; r < kSrftR; ++r) {
        const int64_t lr = hoffs[r + 1] - hoffs[r];
        if (lr == 0) continue;
        int S = zgemm_ksplit(lr, m1, n / 8, num_sms);
        if ((size_t)S * lr * nc > splitk_elems) S = 1;
        e = zgemm_ordered(Wg + hoffs[r], l, Z + (int64_t)r * m1 * nc, m1, Yg + hoffs[r], l, lr,
                          nc, m1, 0, 0.0, 0, 0, st, S, splitk);
        if (e != cudaSuccess) return e;
        *launches += S > 1 ? 2 : 1;
      }
    }
    int64_t sb = (l * nc + 255) / 256;
    if (sb > 8192) sb = 8192;
    k_srft_scatter<<<(unsigned)sb, 256, 0, st>>>(Yg, order, l, nc, Y + c0 * ldy, ldy);
    *launches += 1;
  }
  return cudaGetLastError();
}

}  // namespace rid

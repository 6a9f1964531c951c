// k_zgemm_tma.cu — the ordered complex GEMM of k_zgemm.cu (real embedding, one ascending fma
// chain per output over the real K index: bit-identical to the oracle's loops, docs/RNG.md §5-§6)
// with its operands moved by the Tensor Memory Accelerator, for the tall products: the generation
// A = X·Y0 + ε·E (Mout = m, K = k) and the QR's panel update C −= V·F.
//
// Same fragments as k_zgemm.cu (MMA M = column j of Bm, N = real row r̃ = 2r + {re, im} of the
// 2×2-block expansion R̃ of Rm, K = real index; each lane's accumulator pair is one complex
// output), same per-warp tiles, different staging:
//   - per stage one thread issues one box of Bm (8 complex K = 128 B × BJ columns) and BRC/8 boxes
//     of Rm (8 complex rows = 128 B × 8 complex K), SWIZZLE_128B, with one arrive.expect_tx;
//     out-of-range rows / columns / K are zero-filled by the TMA unit (a zero term leaves every
//     chain unchanged, as the cp.async kernel's zero-fill does);
//   - warps wait on the stage's "full" mbarrier and release it with one arrive on "empty"; only
//     the producing thread waits for "empty" (no __syncthreads per stage);
//   - bank conflicts: the 128-byte swizzle puts 16-byte chunk c of box row ρ at c ^ (ρ mod 8).
//     Bm: lane (g, t) reads column πB(g), real K 4kk + t (chunk 2kk + t/2); with
//     πB(g) = 2(g mod 4) + g/4 the four columns of a half-warp differ in bits 1-2, so their chunk
//     pairs are disjoint (two wavefronts per LDS.64 warp-wide, the minimum). Rm: lane reads complex
//     row q = g/2 + 4(f mod 2) of box f/2 at complex K kr = 2kk + t/2; the row is stored at
//     ρ(q) = 2(q mod 4) + q/4, so the two K rows of a half-warp (kr even / odd) land on disjoint
//     chunk sets. Both permutations are undone in the epilogue.
#include <cstdlib>

#include "rid_device.cuh"
#include "rid_internal.h"
#include "rid_tma.cuh"

namespace rid {

struct ZtmaEpilogue {
  int mode;  // 0: C = acc; 1: C = fma(noise, E(i, col0 + j), acc); 2: C = C − acc
  double noise;
  uint64_t seed;
  int64_t col0;
};

template <int FJ, int FR, int WJ, int WR, int STAGES>
struct ZTCfg {
  static constexpr int kWarps = WJ * WR;
  static constexpr int kThreads = kWarps * 32;
  static constexpr int BJ = WJ * FJ * 8;   // columns per CTA
  static constexpr int BRC = WR * FR * 4;  // complex rows per CTA
  static constexpr int BKC = 8;            // complex K per stage
  static constexpr int kBBox = 128 * BJ;   // bytes: 8 complex K x BJ columns
  static constexpr int kRBox = 128 * BKC;  // bytes: 8 complex rows x BKC K
  static constexpr int kNR = BRC / 8;
  static constexpr int kStage = kBBox + kNR * kRBox;
  static constexpr size_t kSmem = (size_t)STAGES * kStage + 1024;  // + alignment slack
  static_assert(FR % 2 == 0, "fragments in box pairs");
  static_assert(kBBox % 1024 == 0 && kRBox % 1024 == 0, "1 KB box alignment");
};

template <int FJ, int FR, int WJ, int WR, int STAGES, int MINB>
__global__ void __launch_bounds__(WJ* WR * 32, MINB)
    k_zgemm_tma(const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapR,
                double2* __restrict__ C, int64_t ldc, int64_t Mout, int64_t N, int64_t K,
                ZtmaEpilogue ep) {
  using Cf = ZTCfg<FJ, FR, WJ, WR, STAGES>;
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  unsigned char* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wj = warp % WJ, wr = warp / WJ;
  const int r0c = (int)blockIdx.x * Cf::BRC;
  const int64_t j0 = (int64_t)blockIdx.y * Cf::BJ;
  const int nk = (int)((K + Cf::BKC - 1) / Cf::BKC);

  if (tid == 0) {
    tma_prefetch_map(&mapB);
    tma_prefetch_map(&mapR);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cf::kWarps);
    }
    mbar_init_fence();
  }
  __syncthreads();
  auto issue = [&](int kt) {  // thread 0
    const int s = kt % STAGES;
    unsigned char* st = sm + (size_t)s * Cf::kStage;
    const int kc0 = kt * Cf::BKC;
    mbar_expect_tx(&full[s], Cf::kStage);
    tma_box_g2s(st, &mapB, 2 * kc0, (int)j0, &full[s]);
#pragma unroll
    for (int b = 0; b < Cf::kNR; ++b)
      tma_box_g2s(st + Cf::kBBox + b * Cf::kRBox, &mapR, 2 * (r0c + 8 * b), kc0, &full[s]);
  };
  if (tid == 0)
    for (int kt = 0; kt < STAGES - 1 && kt < nk; ++kt) issue(kt);

  double acc[FJ][FR][2];
#pragma unroll
  for (int a = 0; a < FJ; ++a)
#pragma unroll
    for (int b = 0; b < FR; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int pB = ((g & 3) << 1) | (g >> 2);  // πB(g)
  // Bm: row = column (wj FJ 8 + fa 8 + πB(g)), chunk (2kk + t/2) ^ πB(g), word t & 1
  const int bRow = (wj * FJ * 8 + pB) * 128 + (t & 1) * 8;
  const int bc0 = (t >> 1) ^ pB;  // chunk (2kk + t/2) ^ πB(g) = 2kk ^ bc0
  // Rm: fragment f -> box wr FR/2 + f/2, logical row q = g/2 + 4 (f & 1), stored at ρ(q)
  const int comp = (g & 1) ^ (t & 1);
  const unsigned long long sgn = ((g & 1) == 0 && (t & 1) == 1) ? 0x8000000000000000ULL : 0ULL;
  const int q0 = g >> 1, q1 = (g >> 1) + 4;
  const int rho0 = ((q0 & 3) << 1) | (q0 >> 2), rho1 = ((q1 & 3) << 1) | (q1 >> 2);
  const int rBase = Cf::kBBox + wr * (FR / 2) * Cf::kRBox + comp * 8;

  for (int kt = 0; kt < nk; ++kt) {
    if (tid == 0) {
      const int kn = kt + STAGES - 1;
      if (kn < nk) {
        if (kn >= STAGES) mbar_wait(&empty[kn % STAGES], ((kn / STAGES) - 1) & 1);
        issue(kn);
      }
    }
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    const unsigned char* st = sm + (size_t)s * Cf::kStage;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // real K 4kk .. 4kk + 3 of the stage's 16
      const int kr = 2 * kk + (t >> 1);  // complex K row of the R box
      const int bchunk = ((2 * kk) ^ bc0) * 16;
      double a[FJ], b[FR];
#pragma unroll
      for (int f = 0; f < FJ; ++f)
        a[f] = *reinterpret_cast<const double*>(st + bRow + f * 1024 + bchunk);
#pragma unroll
      for (int f = 0; f < FR; ++f) {
        const int rho = (f & 1) ? rho1 : rho0;
        const double v = *reinterpret_cast<const double*>(
            st + rBase + (f >> 1) * Cf::kRBox + kr * 128 + ((rho ^ (kr & 7)) * 16));
        b[f] = __longlong_as_double(__double_as_longlong(v) ^ sgn);
      }
#pragma unroll
      for (int fa = 0; fa < FJ; ++fa)
#pragma unroll
        for (int fb = 0; fb < FR; ++fb) dmma8x8x4(acc[fa][fb][0], acc[fa][fb][1], a[fa], b[fb]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // epilogue: lane (g, t) holds column πB(g) and logical row t (+4 for odd fragments) of its box
  auto out_row = [&](int fb) {
    const int q = t + 4 * (fb & 1);
    return (int64_t)r0c + 8 * (wr * (FR / 2) + (fb >> 1)) + (((q & 3) << 1) | (q >> 2));
  };
#pragma unroll
  for (int fa = 0; fa < FJ; ++fa) {
    const int64_t j = j0 + wj * FJ * 8 + fa * 8 + pB;
    if (j >= N) continue;
#pragma unroll
    for (int fb = 0; fb < FR; ++fb) {
      const int64_t r = out_row(fb);
      if (r >= Mout) continue;
      double2 o = make_double2(acc[fa][fb][0], acc[fa][fb][1]);
      if (ep.mode == 2) {
        const double2 c = C[j * ldc + r];
        o = make_double2(__dsub_rn(c.x, o.x), __dsub_rn(c.y, o.y));
      }
      C[j * ldc + r] = o;
    }
  }
  if (ep.mode == 1) {  // A = fma(noise, E, X·Y0), E(i, j) = N(seed, 3, i, col0 + j); rolled pass
#pragma unroll 1
    for (int qq = 0; qq < FJ * FR; ++qq) {
      const int fa = qq / FR, fb = qq % FR;
      const int64_t j = j0 + wj * FJ * 8 + fa * 8 + pB;
      const int64_t r = out_row(fb);
      if (j >= N || r >= Mout) continue;
      double2* cp = C + j * ldc + r;
      const double2 a = *cp;
      const double2 e = rid_normal(ep.seed, 3u, (uint32_t)r, (uint32_t)(ep.col0 + j));
      *cp = make_double2(__fma_rn(ep.noise, e.x, a.x), __fma_rn(ep.noise, e.y, a.y));
    }
  }
}

template <int FJ, int FR, int WJ, int WR, int STAGES, int MINB>
static cudaError_t launch_zt(const double2* Rm, int64_t ldr, const double2* Bm, int64_t ldb,
                             double2* C, int64_t ldc, int64_t Mout, int64_t N, int64_t K,
                             const ZtmaEpilogue& ep, cudaStream_t st) {
  using Cf = ZTCfg<FJ, FR, WJ, WR, STAGES>;
  auto kern = k_zgemm_tma<FJ, FR, WJ, WR, STAGES, MINB>;
  cudaError_t e;
  if ((e = ensure_dyn_smem((const void*)kern, Cf::kSmem)) != cudaSuccess) return e;
  PFN_cuTensorMapEncodeTiled encode;
  if ((e = tensor_map_encoder(&encode)) != cudaSuccess) return e;
  CUtensorMap mapB, mapR;
  const cuuint32_t estr[2] = {1u, 1u};
  {
    const cuuint64_t gdim[2] = {(cuuint64_t)(2 * K), (cuuint64_t)N};
    const cuuint64_t gstr[1] = {(cuuint64_t)ldb * sizeof(double2)};
    const cuuint32_t box[2] = {16u, (cuuint32_t)Cf::BJ};
    if (encode(&mapB, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)Bm, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t gdim[2] = {(cuuint64_t)(2 * Mout), (cuuint64_t)K};
    const cuuint64_t gstr[1] = {(cuuint64_t)ldr * sizeof(double2)};
    const cuuint32_t box[2] = {16u, (cuuint32_t)Cf::BKC};
    if (encode(&mapR, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)Rm, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int64_t tiles_r = (Mout + Cf::BRC - 1) / Cf::BRC;
  const int64_t tiles_j = (N + Cf::BJ - 1) / Cf::BJ;
  if (tiles_r > 0x7FFFFFFF || tiles_j > 65535 || 2 * Mout > INT32_MAX)
    return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)tiles_r, (unsigned)tiles_j);
  kern<<<grid, Cf::kThreads, Cf::kSmem, st>>>(mapB, mapR, C, ldc, Mout, N, K, ep);
  return cudaGetLastError();
}

// Opt-in (RID_ZGEMM_TMA=1): measured no faster than the cp.async kernel for the generation
// (C3 11.23 vs 11.31 ms, C4 148.6 vs 146.1, C5 316.0 vs 315.3; tools/gen_time.py) — unlike the
// sketch, the generation's short K (k = 128..512 per output tile) leaves no barrier time to win;
// its DMMA loop is bound by the 4-product fragment loads (9 LDS per 8 DMMA). Kept, tested
// bitwise, as the measured alternative.
bool zgemm_tma_enabled() {
  const char* v = select_env("RID_ZGEMM_TMA");
  return v && atoi(v) != 0;
}

// The generation tile of k_zgemm.cu (64 columns x 32 complex rows, 8 warps along j, 3 CTAs per
// SM), 6 stages of 12 KB; RID_ZGEMM_TMA_STAGES = 4 / 8 for depth experiments.
cudaError_t zgemm_tma_ordered(const double2* Rm, int64_t ldr, const double2* Bm, int64_t ldb,
                              double2* C, int64_t ldc, int64_t Mout, int64_t N, int64_t K,
                              int mode, double noise, uint64_t seed, int64_t col0,
                              cudaStream_t st) {
  if (Mout <= 0 || N <= 0) return cudaSuccess;
  const ZtmaEpilogue ep{mode, noise, seed, col0};
  int stages = 6;
  if (const char* v = experiment_env("RID_ZGEMM_TMA_STAGES")) stages = atoi(v);
  if (mode == 2) return launch_zt<1, 8, 8, 1, 2, 3>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st);
  switch (stages) {
    case 4: return launch_zt<1, 8, 8, 1, 4, 3>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st);
    case 8: return launch_zt<1, 8, 8, 1, 8, 2>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st);
    default: return launch_zt<1, 8, 8, 1, 6, 3>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st);
  }
}

}  // namespace rid

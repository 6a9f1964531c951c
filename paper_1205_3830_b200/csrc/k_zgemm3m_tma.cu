// k_zgemm3m_tma.cu — the sketch Y = R · A (north_star) as Gauss's three real
// products on DMMA (reading R31 in DESIGN.md; same arithmetic as k_zgemm3m.cu), with the operand
// tiles moved by the Tensor Memory Accelerator and the stages handed over with mbarriers instead
// of cp.async + __syncthreads:
//   - one thread issues, per stage, BKC/8 boxes of A (8 complex K × BJ columns, 128 B rows) and
//     BR/8 boxes of R (8 complex rows × BKC K) with cp.async.bulk.tensor, SWIZZLE_128B, and one
//     arrive.expect_tx on the stage's "full" barrier; out-of-range rows/columns/K are zero-filled
//     by the TMA unit (no predication in the kernel);
//   - every warp waits only for the stage it is about to read ("full") and releases it with one
//     arrive on its "empty" barrier (count = warps); the producing thread waits for "empty" of the
//     slot it refills, so warps are never held at a CTA-wide barrier and drift freely by up to
//     STAGES − 1 stages;
//   - the tiles are dense (no padding: 28 KB per stage instead of 32.8 KB). The 128-byte swizzle
//     puts the 16-byte chunk q of row ρ at chunk q ^ (ρ & 7); fragment row g of an 8-wide group is
//     mapped to the tile's row π(g) = (g >> 1) + 4 (g & 1), so the eight lanes of every LDS.128
//     phase — g ∈ {2h, 2h + 1}, t = 0..3 — read chunks {c ^ π(2h)} ∪ {c ^ π(2h + 1)} = all eight
//     16-byte bank groups: conflict-free. The permutation is undone in the epilogue (lane (g, t)
//     holds column π(g) and rows t, t + 4 of its fragment).
// Each P is the ascending fma chain over the complex K index inside a K slice, exactly as in
// k_zgemm3m.cu: the two kernels give bit-identical Y (tested).
#include <cstdlib>

#include "rid_device.cuh"
#include "rid_internal.h"
#include "rid_tma.cuh"

namespace rid {

template <int FJ, int FR, int WJ, int WR, int STAGES, int RS>
struct Z3T {
  static constexpr int kWarps = WJ * WR;
  static constexpr int kThreads = kWarps * 32;
  static constexpr int BJ = WJ * FJ * 8;     // columns per CTA
  static constexpr int BR = WR * FR * 8;     // complex rows per CTA
  static constexpr int BKC = 16;             // complex K per stage
  static constexpr int kABox = 128 * BJ;     // bytes: 8 complex K (128 B) x BJ columns
  static constexpr int kRBox = 128 * BKC;    // bytes: 8 complex rows (128 B) x BKC K
  static constexpr int kRsBox = 64 * BKC;   // bytes: 8 rows of Re R + Im R (64 B) x BKC K
  static constexpr int kNA = BKC / 8, kNR = BR / 8;
  static constexpr int kStage = kNA * kABox + kNR * kRBox + (RS ? kNR * kRsBox : 0);
  // + alignment slack, except at 4 stages (two CTAs per SM only fit without it: the static
  // barriers put the dynamic base at 1 KB, checked in the kernel)
  static constexpr size_t kSmem = (size_t)STAGES * kStage + (STAGES >= 4 ? 0 : 1024);
  static_assert(kABox % 1024 == 0 && kRBox % 1024 == 0, "boxes must keep 1 KB alignment");
};

// RS = 1: Re R + Im R comes from a precomputed plane (k_rsum), boxes of 8 rows x BKC K without
// swizzle (a lane's 8-byte load: rows t of 64 B, two wavefronts per warp, the minimum)
// ORD: DMMA issue order within a k-step — 0: (fa, fb, p) with volatile asm; 1: p outermost (the
// products that need the Re + Im sums come last); 2: (fa, fb, p), non-volatile; 3: p outermost,
// non-volatile.
template <int FJ, int FR, int WJ, int WR, int STAGES, int MINB, int RS, int ORD = 0>
__global__ void __launch_bounds__(WJ* WR * 32, MINB)
    k_zgemm3m_tma(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapR,
                  const __grid_constant__ CUtensorMap mapS, double2* __restrict__ C, int64_t ldc, int64_t Mout, int64_t N, int64_t K,
                  int64_t kchunk, int64_t zstride, const Z3Batch bt) {
  using Cf = Z3T<FJ, FR, WJ, WR, STAGES, RS>;
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  unsigned char* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  if (STAGES >= 4 && (smem_u32(smraw) & 1023) != 0) __trap();
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int pg = (g >> 1) + 4 * (g & 1);  // π(g)
  const int wj = warp % WJ, wr = warp / WJ;
  const int r0 = (int)blockIdx.x * Cf::BR;  // first output row of the tile
  const int64_t j0 = (int64_t)blockIdx.y * Cf::BJ;
  int rt0 = r0, jt0 = (int)j0, st0 = r0;     // tile origin in the tensor maps (st0: Rs plane)
  int64_t kbeg = 0, kend = K;
  if (bt.n > 0) {  // batched (blockIdx.z = product): row / column offsets into shared maps
    const int z = blockIdx.z;
    Mout = bt.mout[z];
    if (r0 >= Mout) return;
    rt0 += (int)bt.roff[z];
    st0 += (int)bt.soff[z];
    jt0 += (int)bt.boff[z];
    C += bt.coff[z];
  } else {
    kbeg = (int64_t)blockIdx.z * kchunk;
    kend = (kbeg + kchunk < K) ? kbeg + kchunk : K;
    C += (int64_t)blockIdx.z * zstride;
  }
  const int nk = (int)((kend - kbeg + Cf::BKC - 1) / Cf::BKC);

  if (tid == 0) {
    tma_prefetch_map(&mapA);
    tma_prefetch_map(&mapR);
    if (RS) tma_prefetch_map(&mapS);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cf::kWarps);
    }
    mbar_init_fence();
  }
  __syncthreads();

  auto issue = [&](int kt) {  // thread 0 only
    const int s = kt % STAGES;
    unsigned char* st = sm + (size_t)s * Cf::kStage;
    mbar_expect_tx(&full[s], Cf::kStage);
    const int kc0 = (int)(kbeg + (int64_t)kt * Cf::BKC);
#pragma unroll
    for (int b = 0; b < Cf::kNA; ++b)
      tma_box_g2s(st + b * Cf::kABox, &mapA, 2 * kc0 + 16 * b, jt0, &full[s]);
#pragma unroll
    for (int b = 0; b < Cf::kNR; ++b)
      tma_box_g2s(st + Cf::kNA * Cf::kABox + b * Cf::kRBox, &mapR, 2 * (rt0 + 8 * b), kc0, &full[s]);
    if (RS) {
#pragma unroll
      for (int b = 0; b < Cf::kNR; ++b)
        tma_box_g2s(st + Cf::kNA * Cf::kABox + Cf::kNR * Cf::kRBox + b * Cf::kRsBox, &mapS,
                    st0 + 8 * b, kc0, &full[s]);
    }
  };
  if (tid == 0)
    for (int kt = 0; kt < STAGES - 1 && kt < nk; ++kt) issue(kt);

  double acc[FJ][FR][3][2];
#pragma unroll
  for (int a = 0; a < FJ; ++a)
#pragma unroll
    for (int b = 0; b < FR; ++b)
#pragma unroll
      for (int p = 0; p < 3; ++p) acc[a][b][p][0] = acc[a][b][p][1] = 0.0;

  // lane constants: the swizzled chunk of (K offset t [+4 on odd k-steps]) in row π(g)
  const int offE = (t ^ pg) * 16, offO = ((4 + t) ^ pg) * 16;
  const int aRow = (wj * FJ * 8 + pg) * 128;                                // A: row = column
  const int rRow = Cf::kNA * Cf::kABox + wr * FR * Cf::kRBox + t * 128;     // R: row = K index
  const int sRow = Cf::kNA * Cf::kABox + Cf::kNR * Cf::kRBox + wr * FR * Cf::kRsBox + t * 64 +
                   pg * 8;                                                   // Rs: row = K index

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
    for (int kk = 0; kk < Cf::BKC / 4; ++kk) {
      const int off = (kk & 1) ? offO : offE;
      double a[FJ][3], b[FR][3];
#pragma unroll
      for (int f = 0; f < FJ; ++f) {
        const double2 v = *reinterpret_cast<const double2*>(st + (kk >> 1) * Cf::kABox + aRow +
                                                            f * 1024 + off);
        a[f][0] = v.x;
        a[f][1] = v.y;
        a[f][2] = __dadd_rn(v.x, v.y);
      }
#pragma unroll
      for (int f = 0; f < FR; ++f) {
        const double2 v =
            *reinterpret_cast<const double2*>(st + rRow + f * Cf::kRBox + kk * 512 + off);
        b[f][0] = v.x;
        b[f][1] = v.y;
        b[f][2] = RS ? *reinterpret_cast<const double*>(st + sRow + f * Cf::kRsBox + kk * 256)
                     : __dadd_rn(v.x, v.y);
      }
      if (ORD == 0 || ORD == 2) {
#pragma unroll
        for (int fa = 0; fa < FJ; ++fa)
#pragma unroll
          for (int fb = 0; fb < FR; ++fb)
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              if (ORD == 0) dmma8x8x4(acc[fa][fb][p][0], acc[fa][fb][p][1], a[fa][p], b[fb][p]);
              else dmma8x8x4_nv(acc[fa][fb][p][0], acc[fa][fb][p][1], a[fa][p], b[fb][p]);
            }
      } else {
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
          for (int fa = 0; fa < FJ; ++fa)
#pragma unroll
            for (int fb = 0; fb < FR; ++fb) {
              if (ORD == 1) dmma8x8x4(acc[fa][fb][p][0], acc[fa][fb][p][1], a[fa][p], b[fb][p]);
              else dmma8x8x4_nv(acc[fa][fb][p][0], acc[fa][fb][p][1], a[fa][p], b[fb][p]);
            }
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // epilogue: lane (g, t) holds column π(g) and rows t, t + 4 of each 8 x 8 fragment
#pragma unroll
  for (int fa = 0; fa < FJ; ++fa) {
    const int64_t j = j0 + wj * FJ * 8 + fa * 8 + pg;
    if (j >= N) continue;
#pragma unroll
    for (int fb = 0; fb < FR; ++fb) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = r0 + wr * FR * 8 + fb * 8 + t + 4 * h;
        if (r >= Mout) continue;
        const double p1 = acc[fa][fb][0][h], p2 = acc[fa][fb][1][h], p3 = acc[fa][fb][2][h];
        C[j * ldc + r] = make_double2(__dsub_rn(p1, p2), __dsub_rn(__dsub_rn(p3, p1), p2));
      }
    }
  }
}

__global__ void k_splitk_reduce3t(const double2* __restrict__ part, int S, int64_t Mout, int64_t N,
                                  double2* __restrict__ C, int64_t ldc) {
  const int64_t total = Mout * N, zs = Mout * N;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    double2 a = part[q];
    for (int z = 1; z < S; ++z) {
      const double2 b = part[z * zs + q];
      a = make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
    }
    C[(q / Mout) * ldc + q % Mout] = a;
  }
}

// bt (nullable): bt->n products in one launch, product z = rows [roff, roff + mout) of Rm (Rm
// holding Mout rows in all) times columns [boff, boff + N) of Bm (Bm holding Nb columns in all),
// written to C + coff; rows and columns a tile reads past its product are discarded.
template <int FJ, int FR, int WJ, int WR, int STAGES, int MINB, int RS, int ORD = 0>
static cudaError_t launch3t(const double2* Rm, int64_t ldr, const double* Rs, int64_t ldrs,
                            const double2* Bm, int64_t ldb, double2* C, int64_t ldc, int64_t Mout,
                            int64_t N, int64_t K, cudaStream_t st, int S, double2* partial,
                            const Z3Batch* bt = nullptr, int64_t Nb = 0, int64_t Ms = 0) {
  using Cf = Z3T<FJ, FR, WJ, WR, STAGES, RS>;
  auto kern = k_zgemm3m_tma<FJ, FR, WJ, WR, STAGES, MINB, RS, ORD>;
  cudaError_t e;
  if ((e = ensure_dyn_smem((const void*)kern, Cf::kSmem)) != cudaSuccess) return e;
  PFN_cuTensorMapEncodeTiled encode;
  if ((e = tensor_map_encoder(&encode)) != cudaSuccess) return e;
  // A as a (2K doubles) x N matrix, boxes of 16 doubles x BJ columns; R as (2 Mout) x K, boxes
  // of 16 doubles x BKC K; both 128-byte swizzled, out-of-bounds zero-filled
  CUtensorMap mapA, mapR, mapS;
  const cuuint32_t estr[2] = {1u, 1u};
  {
    const cuuint64_t gdim[2] = {(cuuint64_t)(2 * K), (cuuint64_t)(bt ? Nb : N)};
    const cuuint64_t gstr[1] = {(cuuint64_t)ldb * sizeof(double2)};
    const cuuint32_t box[2] = {16u, (cuuint32_t)Cf::BJ};
    if (encode(&mapA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)Bm, gdim, gstr, box, estr,
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
  mapS = mapR;  // unused unless RS
  if (RS) {
    const cuuint64_t gdim[2] = {(cuuint64_t)(Ms > 0 ? Ms : Mout), (cuuint64_t)K};
    const cuuint64_t gstr[1] = {(cuuint64_t)ldrs * sizeof(double)};
    const cuuint32_t box[2] = {8u, (cuuint32_t)Cf::BKC};
    if (!Rs || (ldrs * sizeof(double)) % 16 != 0 ||
        encode(&mapS, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)Rs, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  if (bt) {
    int64_t mmax = 0;
    for (int z = 0; z < bt->n; ++z) mmax = bt->mout[z] > mmax ? bt->mout[z] : mmax;
    const int64_t tr = (mmax + Cf::BR - 1) / Cf::BR, tj = (N + Cf::BJ - 1) / Cf::BJ;
    if (tr < 1 || tj > 65535 || Mout > INT32_MAX / 2 || Nb > INT32_MAX)
      return cudaErrorInvalidConfiguration;
    dim3 grid((unsigned)tr, (unsigned)tj, (unsigned)bt->n);
    kern<<<grid, Cf::kThreads, Cf::kSmem, st>>>(mapA, mapR, mapS, C, ldc, Mout, N, K, K, 0, *bt);
    return cudaGetLastError();
  }
  const int64_t tiles_r = (Mout + Cf::BR - 1) / Cf::BR;
  const int64_t tiles_j = (N + Cf::BJ - 1) / Cf::BJ;
  int64_t kc = K > 0 ? K : 1;
  double2* Cout = C;
  int64_t ldo = ldc, zs = 0;
  if (S > 1 && partial) {
    kc = (K + S - 1) / S;
    kc = ((kc + Cf::BKC - 1) / Cf::BKC) * Cf::BKC;
    S = (int)((K + kc - 1) / kc);
    if (S > 1) {
      Cout = partial;
      ldo = Mout;
      zs = Mout * N;
    }
  } else {
    S = 1;
  }
  if (tiles_r > 65535 || tiles_j > 65535 || S > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)tiles_r, (unsigned)tiles_j, (unsigned)S);
  Z3Batch none{};
  kern<<<grid, Cf::kThreads, Cf::kSmem, st>>>(mapA, mapR, mapS, Cout, ldo, Mout, N, K, kc, zs, none);
  e = cudaGetLastError();
  if (e != cudaSuccess || S == 1) return e;
  int64_t blocks = (Mout * N + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_splitk_reduce3t<<<(unsigned)blocks, 256, 0, st>>>(partial, S, Mout, N, C, ldc);
  return cudaGetLastError();
}

// The TMA pipeline covers all three tiles — 48 rows (C3, C4), 40 (C2, C5; with the Re R + Im R
// plane when one is passed), 24 (C1) — unless RID_Z3_TMA=0.
bool zgemm3m_tma_enabled(int64_t Mout) {
  const char* v = select_env("RID_Z3_TMA");
  return !(v && atoi(v) == 0) && Mout > 0;
}

cudaError_t zgemm3m_tma(const double2* Rm, int64_t ldr, const double* Rs, int64_t ldrs,
                        const double2* Bm, int64_t ldb, double2* C, int64_t ldc, int64_t Mout,
                        int64_t N, int64_t K, cudaStream_t st, int ksplit, double2* partial) {
  if (Mout <= 0 || N <= 0) return cudaSuccess;
#define RID_L3T(...) \
  launch3t<__VA_ARGS__>(Rm, ldr, Rs, ldrs, Bm, ldb, C, ldc, Mout, N, K, st, ksplit, partial)
  int var = 0;
  if (const char* v = select_env("RID_Z3T_VARIANT")) var = atoi(v);  // pipeline-depth experiments
  if (zgemm3m_tile_rows(Mout) == 40) {
    if (!Rs) return RID_L3T(1, 5, 8, 1, 3, 2, 0);
    switch (var) {
      case 2: return RID_L3T(1, 5, 8, 1, 2, 2, 1);
      case 11: return RID_L3T(1, 5, 8, 1, 3, 2, 1, 1);
      case 12: return RID_L3T(1, 5, 8, 1, 3, 2, 1, 2);
      case 13: return RID_L3T(1, 5, 8, 1, 3, 2, 1, 3);
      default: return RID_L3T(1, 5, 8, 1, 3, 2, 1);
    }
  }
  if (zgemm3m_tile_rows(Mout) == 24)
    return Rs ? RID_L3T(1, 3, 8, 1, 3, 2, 1) : RID_L3T(1, 3, 8, 1, 3, 2, 0);
  // 48 rows: with the Re R + Im R plane (3 of the 5 adds per k-step gone from the FP64 pipe the
  // DMMAs share) and 2 stages: C4 103.0 -> 100.5 ms (3 stages 101.3); sums in registers otherwise
  switch (var) {
    case 2: return RID_L3T(2, 3, 4, 2, 2, 2, 0);
    case 3: return RID_L3T(2, 3, 4, 2, 3, 2, 0);
    case 4: return RID_L3T(2, 3, 4, 2, 4, 2, 0);
    case 30: if (Rs) return RID_L3T(2, 3, 4, 2, 3, 2, 1); break;
    case 11: return RID_L3T(2, 3, 4, 2, 3, 2, 0, 1);
    case 12: return RID_L3T(2, 3, 4, 2, 3, 2, 0, 2);
    case 13: return RID_L3T(2, 3, 4, 2, 3, 2, 0, 3);
    default: break;
  }
  return Rs ? RID_L3T(2, 3, 4, 2, 2, 2, 1) : RID_L3T(2, 3, 4, 2, 3, 2, 0);
#undef RID_L3T
}

// One tile height forced (48 / 40 / 32 / 24 rows), with the Re R + Im R plane when given: the two
// parts of a row-split sketch (sketch_gemm)
cudaError_t zgemm3m_tma_rows(const double2* Rm, int64_t ldr, const double* Rs, int64_t ldrs,
                             const double2* Bm, int64_t ldb, double2* C, int64_t ldc, int64_t Mout,
                             int64_t N, int64_t K, cudaStream_t st, int ksplit, double2* partial,
                             int rows) {
  if (Mout <= 0 || N <= 0) return cudaSuccess;
#define RID_L3T(...) \
  launch3t<__VA_ARGS__>(Rm, ldr, Rs, ldrs, Bm, ldb, C, ldc, Mout, N, K, st, ksplit, partial)
  switch (rows) {
    case 48: return Rs ? RID_L3T(2, 3, 4, 2, 2, 2, 1) : RID_L3T(2, 3, 4, 2, 3, 2, 0);
    case 40: return Rs ? RID_L3T(1, 5, 8, 1, 3, 2, 1) : RID_L3T(1, 5, 8, 1, 3, 2, 0);
    case 32: return Rs ? RID_L3T(2, 2, 4, 2, 2, 2, 1) : RID_L3T(2, 2, 4, 2, 3, 2, 0);
    case 24: return Rs ? RID_L3T(1, 3, 8, 1, 3, 2, 1) : RID_L3T(1, 3, 8, 1, 3, 2, 0);
    default: return cudaErrorInvalidValue;
  }
#undef RID_L3T
}

// The SRFT's residue products (k_srft.cu): bt.roff = first row of product z in Rm (Mtot rows in
// all), bt.boff = ELEMENT offset of its B block in Bm (a multiple of ldb: the block starts at
// column boff / ldb of the Nb = nblk * N columns), bt.coff / bt.mout as for zgemm3m_batched.
cudaError_t zgemm3m_tma_batched(const double2* Rm, int64_t ldr, int64_t Mtot, const double2* Bm,
                                int64_t ldb, int64_t Nb, double2* C, int64_t ldc,
                                const Z3Batch& bt, int64_t N, int64_t K, cudaStream_t st) {
  return zgemm3m_tma_batched_h(Rm, ldr, Mtot, Bm, ldb, Nb, C, ldc, bt, N, K, 0, st, nullptr, 0, 0);
}

// rows = 48 / 40 / 24 forces the tile height; 0 picks it from the largest product
cudaError_t zgemm3m_tma_batched_h(const double2* Rm, int64_t ldr, int64_t Mtot, const double2* Bm,
                                  int64_t ldb, int64_t Nb, double2* C, int64_t ldc,
                                  const Z3Batch& bt, int64_t N, int64_t K, int rows,
                                  cudaStream_t st, const double* Rs, int64_t ldrs, int64_t Ms) {
  if (bt.n <= 0 || N <= 0) return cudaSuccess;
  Z3Batch b = bt;
  for (int z = 0; z < b.n; ++z) {
    if (b.boff[z] % ldb) return cudaErrorInvalidValue;
    b.boff[z] /= ldb;
  }
  int64_t mmax = 0;
  for (int z = 0; z < b.n; ++z) mmax = b.mout[z] > mmax ? b.mout[z] : mmax;
  // with a Re + Im plane of Rm (Rs: Ms rows, product z from row soff[z], even): the sums come
  // from shared memory
  const char* v = select_env("RID_Z3_BATCH_RS");
  bool rs = Rs && !(v && atoi(v) == 0);
  for (int z = 0; z < b.n && rs; ++z)
    if (b.soff[z] & 1) return cudaErrorInvalidValue;
#define RID_LB(FJ, FR, WJ, WR, ST, RS) \
  launch3t<FJ, FR, WJ, WR, ST, 2, RS>(Rm, ldr, Rs, ldrs, Bm, ldb, C, ldc, Mtot, N, K, st, 1, \
                                      nullptr, &b, Nb, Ms)
  switch (rows ? rows : zgemm3m_tile_rows(mmax)) {
    case 48: return rs ? RID_LB(2, 3, 4, 2, 2, 1) : RID_LB(2, 3, 4, 2, 3, 0);
    case 40: return rs ? RID_LB(1, 5, 8, 1, 3, 1) : RID_LB(1, 5, 8, 1, 3, 0);
    default:  // 24 rows (the residues' l/16 rows at C2, C3)
      return rs ? RID_LB(1, 3, 8, 1, 3, 1) : RID_LB(1, 3, 8, 1, 3, 0);
  }
#undef RID_LB
}

}  // namespace rid

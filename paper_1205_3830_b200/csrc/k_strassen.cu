// k_strassen.cu — the sketch Y = R · A (north_star) with ONE level of Strassen's
// algorithm on top of Gauss's three real products (reading R32): seven half-size
// products instead of eight, so the tensor pipe executes 7/8 · 6 l m n = 5.25 l m n flop against
// the metric's 8 l m n.
//
// The 2 x 2 block split (every pairing is a fixed function of global indices):
//   rows    r < l/2  |  r >= l/2                       (R, Y: row halves; l % 4 == 0)
//   K       k < m/2  |  k >= m/2                       (R columns, A rows; m % 32 == 0)
//   columns bit 5 of the column index: the two 32-column halves of every 64-column group of A
//           (and Y) — a pairing that stays inside every 64-aligned column shard, so any G-way
//           sharding (n / G a multiple of 64) reproduces the whole matrix's bits.
// With R_ab (row half a, K half b) and A_bc (K half b, column half c):
//   M1 = (R11 + R22)(A11 + A22)   M2 = (R21 + R22) A11   M3 = R11 (A12 - A22)
//   M4 = R22 (A21 - A11)           M5 = (R11 + R12) A22   M6 = (R21 - R11)(A11 + A12)
//   M7 = (R12 - R22)(A21 + A22)
//   Y11 = ((M1 + M4) - M5) + M7   Y12 = M3 + M5   Y21 = M2 + M4   Y22 = ((M1 - M2) + M3) + M6
// The R combinations (l m / 4 complex each) are formed once per call by k_strassen_rcomb, with
// their Re + Im planes; the A combinations are formed in the fragment loads of the product kernel
// (two TMA-staged A tiles per stage, one DFMA per component: fma(+-1, a2, a1) is the exact sum or
// difference), so A is still only read, never rewritten (16 GiB at C4). Each product is the
// k_zgemm3m_tma pipeline: TMA boxes with 128-byte swizzle, mbarrier full/empty ring, DMMA.8x8x4,
// the same conflict-free lane permutation. The seven products run as one launch (blockIdx.z),
// into a workspace M (7 x l/2 x n/2), combined into Y by k_strassen_combine.
#include <cstdlib>
#include <type_traits>

#include "rid_device.cuh"
#include "rid_internal.h"
#include "rid_tma.cuh"

namespace rid {

// A terms of product z: (K half, column half) of term 1 and term 2, sign of term 2 (0: none)
__constant__ int c_strassen_a[7][5] = {
    {0, 0, 1, 1, 1},   // M1: A11 + A22
    {0, 0, 0, 0, 0},   // M2: A11
    {0, 1, 1, 1, -1},  // M3: A12 - A22
    {1, 0, 0, 0, -1},  // M4: A21 - A11
    {1, 1, 0, 0, 0},   // M5: A22
    {0, 0, 0, 1, 1},   // M6: A11 + A12
    {1, 0, 1, 1, 1},   // M7: A21 + A22
};
// R terms of product z: (row half, K half) of term 1 and term 2, sign of term 2 (0: none)
__constant__ int c_strassen_r[7][5] = {
    {0, 0, 1, 1, 1},   // M1: R11 + R22
    {1, 0, 1, 1, 1},   // M2: R21 + R22
    {0, 0, 0, 0, 0},   // M3: R11
    {1, 1, 0, 0, 0},   // M4: R22
    {0, 0, 0, 1, 1},   // M5: R11 + R12
    {1, 0, 0, 0, -1},  // M6: R21 - R11
    {0, 1, 1, 1, -1},  // M7: R12 - R22
};

// Rc (7 lh rows x mh, ld ldc: product z in rows [z lh, (z + 1) lh)) and Rs = Re Rc + Im Rc
// (ld lds, pad rows zero) from R (l x m, ld ldr). One thread per (row, K) of a product.
__global__ void k_strassen_rcomb(const double2* __restrict__ R, int64_t ldr, int lh, int64_t mh,
                                 double2* __restrict__ Rc, int64_t ldc, double* __restrict__ Rs,
                                 int64_t lds) {
  const int64_t rows = 7 * (int64_t)lh, total = lds * mh;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = q / lds, rr = q - k * lds;
    if (rr >= rows) {
      Rs[q] = 0.0;
      continue;
    }
    const int z = (int)(rr / lh), r = (int)(rr - (int64_t)z * lh);
    const int* t = c_strassen_r[z];
    double2 v = R[(t[1] * mh + k) * ldr + t[0] * lh + r];
    if (t[4] != 0) {
      const double2 w = R[(t[3] * mh + k) * ldr + t[2] * lh + r];
      v = t[4] > 0 ? make_double2(__dadd_rn(v.x, w.x), __dadd_rn(v.y, w.y))
                   : make_double2(__dsub_rn(v.x, w.x), __dsub_rn(v.y, w.y));
    }
    Rc[k * ldc + rr] = v;
    Rs[q] = __dadd_rn(v.x, v.y);
  }
}

// Y (l x ncols block, ld ldy) from M (S K slices of 7 products of lh x nh, ld lh, product stride
// lh nh, slice stride 7 lh nh): each product's slices added in slice order, then combined
__global__ void k_strassen_combine(const double2* __restrict__ M, int lh, int64_t nh, int S,
                                   double2* __restrict__ Y, int64_t ldy) {
  const int64_t total = (int64_t)lh * nh, zs = total, ss = 7 * total;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = q / lh;
    const int r = (int)(q - c * lh);
    double2 mz[7];
#pragma unroll
    for (int z = 0; z < 7; ++z) {
      double2 a = M[z * zs + q];
      for (int s = 1; s < S; ++s) {
        const double2 b = M[s * ss + z * zs + q];
        a = make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
      }
      mz[z] = a;
    }
    const double2 m1 = mz[0], m2 = mz[1], m3 = mz[2], m4 = mz[3];
    const double2 m5 = mz[4], m6 = mz[5], m7 = mz[6];
    double2 y11, y12, y21, y22;
    y11.x = __dadd_rn(__dsub_rn(__dadd_rn(m1.x, m4.x), m5.x), m7.x);
    y11.y = __dadd_rn(__dsub_rn(__dadd_rn(m1.y, m4.y), m5.y), m7.y);
    y12.x = __dadd_rn(m3.x, m5.x);
    y12.y = __dadd_rn(m3.y, m5.y);
    y21.x = __dadd_rn(m2.x, m4.x);
    y21.y = __dadd_rn(m2.y, m4.y);
    y22.x = __dadd_rn(__dadd_rn(__dsub_rn(m1.x, m2.x), m3.x), m6.x);
    y22.y = __dadd_rn(__dadd_rn(__dsub_rn(m1.y, m2.y), m3.y), m6.y);
    // half-column c of column half h -> block column (c / 32) 64 + 32 h + c % 32
    const int64_t c0 = (c >> 5) * 64 + (c & 31), c1 = c0 + 32;
    Y[c0 * ldy + r] = y11;
    Y[c1 * ldy + r] = y12;
    Y[c0 * ldy + lh + r] = y21;
    Y[c1 * ldy + lh + r] = y22;
  }
}

__device__ __forceinline__ void tma_box4_g2s(void* dst, const CUtensorMap* map, int x, int y,
                                             int z, int w, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(b))
      : "memory");
}

template <int FJ, int FR, int WJ, int WR, int STAGES, int BK = 16>
struct SCfg {
  static constexpr int kWarps = WJ * WR;
  static constexpr int kThreads = kWarps * 32;
  static constexpr int BJ = WJ * FJ * 8;     // half-columns per CTA (64: two 32-column boxes)
  static constexpr int BR = WR * FR * 8;     // product rows per CTA
  static constexpr int BKC = BK;             // complex K per stage (8 or 16)
  static constexpr int kABox = 128 * BJ;     // 8 complex K x BJ half-columns (BJ / 64 TMA boxes)
  static constexpr int kRBox = 128 * BKC;    // 8 complex rows x BKC K
  static constexpr int kRsBox = 64 * BKC;    // 8 rows of Re + Im x BKC K
  static constexpr int kNA = BKC / 8, kNR = BR / 8;
  static constexpr int kAterm = kNA * kABox;
  static constexpr int kStage = 2 * kAterm + kNR * kRBox + kNR * kRsBox;
  static constexpr size_t kSmem = (size_t)STAGES * kStage + 1024;
  static_assert(BJ % 64 == 0, "a tile is whole pairs of 32-column groups of one column half");
  static_assert(kABox % 1024 == 0 && kRBox % 1024 == 0 && kStage % 1024 == 0,
                "boxes and stages keep 1 KB alignment (128-byte swizzle)");
};

// One launch computes rows [rbeg, rend) of the products selected by blockIdx.z: TWO = the
// products whose A operand is a sum or difference of two blocks (M1, M3, M4, M6, M7), else the
// two with a single block (M2, M5) — separate instantiations, so neither carries the other's
// registers. mapA: the A block as 4D (2m doubles, 32 columns, 2 halves, n/64 groups); mapR /
// mapS: Rc / Rs.
template <int FJ, int FR, int WJ, int WR, int STAGES, int MINB, bool TWO, int BK>
__global__ void __launch_bounds__(WJ* WR * 32, MINB)
    k_strassen3m(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapR,
                 const __grid_constant__ CUtensorMap mapS, double2* __restrict__ M, int lh,
                 int64_t nh, int mh, int rbeg, int rend, int raster, int kslice) {
  using Cf = SCfg<FJ, FR, WJ, WR, STAGES, BK>;
  extern __shared__ __align__(1024) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  unsigned char* sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int pg = (g >> 1) + 4 * (g & 1);  // π(g), as in k_zgemm3m_tma.cu
  const int wj = warp % WJ, wr = warp / WJ;
  // raster 0: blockIdx = (row tile, column tile, product); raster 1: blockIdx.x = product +
  // nz * row tile, so every product of a column tile runs at once and they share its A tiles in L2
  constexpr int nz = TWO ? 5 : 2;
  // the tile (product z, first product row, first half-column), recomputed from blockIdx where
  // used so no index is live across the K loop (the loop runs at the 128-register limit)
  auto tile_z = [&]() -> int {
    const int zi = raster ? (int)(blockIdx.x % nz) : (int)blockIdx.z;
    return TWO ? (int)((0x65320u >> (4 * zi)) & 15u)  // M1 M3 M4 M6 M7
               : (zi ? 4 : 1);                         // M2 M5
  };
  auto tile_r0 = [&]() -> int {
    return rbeg + (int)(raster ? blockIdx.x / nz : blockIdx.x) * Cf::BR;
  };
  // sign of the second A term as a mask on the high word: v - w = v + (w with its sign flipped),
  // an integer XOR off the FP64 pipe, then one DADD (the exact sum / difference, one rounding)
  const unsigned sgmask = c_strassen_a[tile_z()][4] < 0 ? 0x80000000u : 0u;
  constexpr bool two = TWO;
  // K slice blockIdx.z (raster 1; the launcher forces it when there are slices): complex K
  // [kbeg, kbeg + kslice) of the product's m/2, its partial product to slice z of M
  const int kbeg = raster ? (int)blockIdx.z * kslice : 0;
  const int kend = raster ? min(mh, kbeg + kslice) : mh;
  const int nk = (kend - kbeg) / Cf::BKC;

  if (tid == 0) {
    tma_prefetch_map(&mapA);
    tma_prefetch_map(&mapR);
    tma_prefetch_map(&mapS);
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cf::kWarps);
    }
    mbar_init_fence();
  }
  __syncthreads();

  auto issue = [&](int kt) {  // thread 0 only (tile coordinates recomputed: short live ranges)
    const int zz = tile_z();
    const int grp = (int)(blockIdx.y * (Cf::BJ / 32));  // the tile's first 64-column group
    const int rrow = zz * lh + tile_r0();                // the tile's first row in Rc / Rs
    const int kh1 = c_strassen_a[zz][0], h1 = c_strassen_a[zz][1];
    const int kh2 = c_strassen_a[zz][2], h2 = c_strassen_a[zz][3];
    const int s = kt % STAGES;
    unsigned char* st = sm + (size_t)s * Cf::kStage;
    mbar_expect_tx(&full[s], two ? Cf::kStage : Cf::kStage - Cf::kAterm);
    const int kc0 = kbeg + kt * Cf::BKC;
#pragma unroll
    for (int b = 0; b < Cf::kNA; ++b)
#pragma unroll
      for (int i = 0; i < Cf::BJ / 64; ++i) {  // one 4D box = 64 half-columns (two groups)
        tma_box4_g2s(st + b * Cf::kABox + i * 8192, &mapA, 2 * (kh1 * mh + kc0) + 16 * b, 0, h1,
                     grp + 2 * i, &full[s]);
        if (two)
          tma_box4_g2s(st + Cf::kAterm + b * Cf::kABox + i * 8192, &mapA,
                       2 * (kh2 * mh + kc0) + 16 * b, 0, h2, grp + 2 * i, &full[s]);
      }
#pragma unroll
    for (int b = 0; b < Cf::kNR; ++b)
      tma_box_g2s(st + 2 * Cf::kAterm + b * Cf::kRBox, &mapR, 2 * (rrow + 8 * b), kc0, &full[s]);
#pragma unroll
    for (int b = 0; b < Cf::kNR; ++b)
      tma_box_g2s(st + 2 * Cf::kAterm + Cf::kNR * Cf::kRBox + b * Cf::kRsBox, &mapS,
                  rrow + 8 * b, kc0, &full[s]);
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

  const int offE = (t ^ pg) * 16, offO = ((4 + t) ^ pg) * 16;
  const int aRow = (wj * FJ * 8 + pg) * 128;
  const int rRow = 2 * Cf::kAterm + wr * FR * Cf::kRBox + t * 128;
  const int sRow = 2 * Cf::kAterm + Cf::kNR * Cf::kRBox + wr * FR * Cf::kRsBox + t * 64 + pg * 8;

  auto kstep = [&](const unsigned char* st, auto TWO) {
#pragma unroll
    for (int kk = 0; kk < Cf::BKC / 4; ++kk) {
      const int off = (kk & 1) ? offO : offE;
      double a[FJ][3], b[FR][3];
#pragma unroll
      for (int f = 0; f < FJ; ++f) {
        const unsigned char* pa = st + (kk >> 1) * Cf::kABox + aRow + f * 1024 + off;
        double2 v = *reinterpret_cast<const double2*>(pa);
        if constexpr (decltype(TWO)::value) {
          const double2 w = *reinterpret_cast<const double2*>(pa + Cf::kAterm);
          v.x = __dadd_rn(v.x, __hiloint2double(__double2hiint(w.x) ^ (int)sgmask,
                                                __double2loint(w.x)));
          v.y = __dadd_rn(v.y, __hiloint2double(__double2hiint(w.y) ^ (int)sgmask,
                                                __double2loint(w.y)));
        }
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
        b[f][2] = *reinterpret_cast<const double*>(st + sRow + f * Cf::kRsBox + kk * 256);
      }
#pragma unroll
      for (int fa = 0; fa < FJ; ++fa)
#pragma unroll
        for (int fb = 0; fb < FR; ++fb)
#pragma unroll
          for (int p = 0; p < 3; ++p)
            dmma8x8x4(acc[fa][fb][p][0], acc[fa][fb][p][1], a[fa][p], b[fb][p]);
    }
  };

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
    kstep(st, std::integral_constant<bool, TWO>{});
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // epilogue: lane (g, t) holds half-column π(g) and rows t, t + 4 of each 8 x 8 fragment
  M += (int64_t)tile_z() * lh * nh + (raster ? (int64_t)blockIdx.z * 7 * lh * nh : 0);
  const int r0 = tile_r0();
  const int64_t j0 = (int64_t)blockIdx.y * Cf::BJ;  // first half-column
#pragma unroll
  for (int fa = 0; fa < FJ; ++fa) {
    const int64_t j = j0 + wj * FJ * 8 + fa * 8 + pg;
    if (j >= nh) continue;
#pragma unroll
    for (int fb = 0; fb < FR; ++fb) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = r0 + wr * FR * 8 + fb * 8 + t + 4 * h;
        if (r >= rend) continue;
        const double p1 = acc[fa][fb][0][h], p2 = acc[fa][fb][1][h], p3 = acc[fa][fb][2][h];
        M[j * lh + r] = make_double2(__dsub_rn(p1, p2), __dsub_rn(__dsub_rn(p3, p1), p2));
      }
    }
  }
}

// ------------------------------------------------------------------------------- host side --
bool strassen_enabled() {
  const char* v = select_env("RID_SKETCH_STRASSEN");  // 0: the plain 3M sketch (tests)
  return !(v && atoi(v) == 0);
}

// The plan is a function of (l, m, n) only (G-invariance): l % 4 == 0 (even row halves), l >= 64,
// m % 32 == 0 (whole stages per K half), m >= 1024, n % 512 == 0 — C2 to C5; K slices
// (strassen_ksplit) where the 3M plan would split K too (C2, C3).
// The tile height of a product's rows: 48 (the remainder on its own height), or the smallest of
// 24 / 32 / 40 that holds l/2 < 48 rows (C2: 40)
static int strassen_main_rows(int64_t lh) {
  if (lh >= 48) return 48;
  return lh <= 24 ? 24 : lh <= 32 ? 32 : 40;
}

bool strassen_plan(int64_t l, int64_t m, int64_t n, int num_sms) {
  (void)num_sms;
  if (!strassen_enabled() || sketch_mults() != 3 || !zgemm3m_tma_enabled(l)) return false;
  // n % 512: every G <= 8 that divides n gives 64-aligned shards (the column pairing's groups)
  if (l % 4 != 0 || l < 64 || m % 32 != 0 || m < 1024 || n % 512 != 0) return false;
  if (l / 2 > 0x3FFFFFFF / 7) return false;
  if (const char* v = experiment_env("RID_STR_UNSPLIT_ONLY"))  // round-2 first plan: C4, C5
    if (atoi(v) != 0 && zgemm3m_ksplit(l, m, n / 8, num_sms) != 1) return false;
  return true;
}

// K slices of the Strassen products: enough CTAs for two per SM at the n/8-column shard of an
// 8-GPU run (a function of (l, m, n) only, so every column's bits are independent of the
// sharding), slices of at least 256 complex K, at most 16. C4, C5: 1; C3: 6; C2: 5.
int strassen_ksplit(int64_t l, int64_t m, int64_t n, int num_sms) {
  const int64_t lh = l / 2, mh = m / 2;
  const int64_t h = strassen_main_rows(lh);
  const int64_t rt = (lh + h - 1) / h;
  const int64_t ct = (n / 16 + 63) / 64;  // half-column tiles of the n/8 shard
  const int64_t ctas = 7 * rt * (ct > 0 ? ct : 1);
  int64_t s = (2 * (int64_t)num_sms + ctas - 1) / ctas;
  const int64_t smax = mh / 256 > 1 ? mh / 256 : 1;
  if (s > smax) s = smax;
  if (s > 16) s = 16;
  return s < 1 ? 1 : (int)s;
}

StrassenWs strassen_ws(int64_t l, int64_t m, int64_t ncols) {
  StrassenWs w{};
  const int64_t lh = l / 2, mh = m / 2;
  w.ldc = 7 * lh;
  w.lds = rsum_ld(7 * lh);
  w.rc_bytes = sizeof(double2) * (size_t)w.ldc * mh;
  w.rs_bytes = sizeof(double) * (size_t)w.lds * mh;
  w.m_bytes = sizeof(double2) * (size_t)7 * lh * (ncols / 2);  // per K slice
  return w;
}

cudaError_t strassen_rcomb(const double2* R, int64_t l, int64_t m, int64_t ldr, double2* Rc,
                           int64_t ldc, double* Rs, int64_t lds, cudaStream_t st) {
  const int64_t total = lds * (m / 2);
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_strassen_rcomb<<<(unsigned)blocks, 256, 0, st>>>(R, ldr, (int)(l / 2), m / 2, Rc, ldc, Rs,
                                                     lds);
  return cudaGetLastError();
}

template <int FJ, int FR, int WJ, int WR, int STAGES, int MINB, int BK = 16>
static cudaError_t launch_products(const CUtensorMap& mapA, const double2* Rc, int64_t ldc,
                                   const double* Rs, int64_t lds, double2* M, int lh, int64_t nh,
                                   int64_t mh, int rbeg, int rend, cudaStream_t st, int raster,
                                   int S) {
  using Cf = SCfg<FJ, FR, WJ, WR, STAGES, BK>;
  auto kern2 = k_strassen3m<FJ, FR, WJ, WR, STAGES, MINB, true, BK>;
  auto kern1 = k_strassen3m<FJ, FR, WJ, WR, STAGES, MINB, false, BK>;
  cudaError_t e;
  if ((e = ensure_dyn_smem((const void*)kern2, Cf::kSmem)) != cudaSuccess) return e;
  if ((e = ensure_dyn_smem((const void*)kern1, Cf::kSmem)) != cudaSuccess) return e;
  PFN_cuTensorMapEncodeTiled encode;
  if ((e = tensor_map_encoder(&encode)) != cudaSuccess) return e;
  const cuuint32_t estr[2] = {1u, 1u};
  CUtensorMap mapR, mapS;
  {
    const cuuint64_t gdim[2] = {(cuuint64_t)(2 * 7 * (int64_t)lh), (cuuint64_t)mh};
    const cuuint64_t gstr[1] = {(cuuint64_t)ldc * sizeof(double2)};
    const cuuint32_t box[2] = {16u, (cuuint32_t)Cf::BKC};
    if (encode(&mapR, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)Rc, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t gdim[2] = {(cuuint64_t)(7 * (int64_t)lh), (cuuint64_t)mh};
    const cuuint64_t gstr[1] = {(cuuint64_t)lds * sizeof(double)};
    const cuuint32_t box[2] = {8u, (cuuint32_t)Cf::BKC};
    if (encode(&mapS, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)Rs, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int64_t tr = (rend - rbeg + Cf::BR - 1) / Cf::BR, tj = (nh + Cf::BJ - 1) / Cf::BJ;
  if (tr < 1 || tj > 65535) return cudaErrorInvalidConfiguration;
  if (const char* v = experiment_env("RID_STR_RASTER")) raster = atoi(v);
  if (S > 1) raster = 1;  // blockIdx.z is the K slice
  // complex K per slice: whole stages
  const int kslice = (int)(((mh + S - 1) / S + Cf::BKC - 1) / Cf::BKC * Cf::BKC);
  const dim3 g2 = raster ? dim3((unsigned)(tr * 5), (unsigned)tj, (unsigned)S)
                         : dim3((unsigned)tr, (unsigned)tj, 5u);
  const dim3 g1 = raster ? dim3((unsigned)(tr * 2), (unsigned)tj, (unsigned)S)
                         : dim3((unsigned)tr, (unsigned)tj, 2u);
  kern2<<<g2, Cf::kThreads, Cf::kSmem, st>>>(mapA, mapR, mapS, M, lh, nh, (int)mh, rbeg, rend,
                                             raster, kslice);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  kern1<<<g1, Cf::kThreads, Cf::kSmem, st>>>(mapA, mapR, mapS, M, lh, nh, (int)mh, rbeg, rend,
                                             raster, kslice);
  return cudaGetLastError();
}

// rows = the tile height. The 48-row main part: 8 warps along j (1 x 6 fragments: one A fragment,
// so one A combination, per warp) with the product-major raster (measured, tools/strassen_check.py,
// profiles/r02/s2_strassen_variants.txt: C4 90.7 ms, C5 201.6 ms against 92.1-92.7 / 202.9-203.5
// for 2 x 4 warps or the (row, column, product) raster; RID_STR_TILE / RID_STR_RASTER in an
// experiments build).
static cudaError_t products_rows(int rows, int rem, const CUtensorMap& mapA, const double2* Rc,
                                 int64_t ldc, const double* Rs, int64_t lds, double2* M, int lh,
                                 int64_t nh, int64_t mh, int rbeg, int rend, cudaStream_t st,
                                 int S) {
  (void)rem;
  int tile = 1;
  if (const char* v = experiment_env("RID_STR_TILE")) tile = atoi(v);
  const int raster = 1;
#define RID_LP(...) \
  launch_products<__VA_ARGS__>(mapA, Rc, ldc, Rs, lds, M, lh, nh, mh, rbeg, rend, st, raster, S)
  if (rows == 48 && tile == 1) return RID_LP(1, 6, 8, 1, 2, 2);
  if (rows == 48 && tile == 5) return RID_LP(1, 6, 16, 1, 2, 1);      // 48 x 128, one CTA/SM
  switch (rows) {
    case 48: return RID_LP(2, 3, 4, 2, 2, 2);
    case 40: return RID_LP(1, 5, 8, 1, 2, 2);
    case 32: return RID_LP(2, 2, 4, 2, 2, 2);
    case 24: return RID_LP(1, 3, 8, 1, 2, 2);
    default: return cudaErrorInvalidValue;
  }
#undef RID_LP
}

cudaError_t strassen_sketch(const double2* Rc, int64_t ldc, const double* Rs, int64_t lds,
                            const double2* A, int64_t lda, double2* Y, int64_t ldy, int64_t l,
                            int64_t ncols, int64_t m, double2* M, int S, cudaStream_t st,
                            const SketchAux* aux, int* launches) {
  if (ncols <= 0) return cudaSuccess;
  if (l % 4 || m % 32 || ncols % 64 || S < 1) return cudaErrorInvalidValue;
  const int lh = (int)(l / 2);
  const int64_t mh = m / 2, nh = ncols / 2;
  cudaError_t e;
  PFN_cuTensorMapEncodeTiled encode;
  if ((e = tensor_map_encoder(&encode)) != cudaSuccess) return e;
  // A block as (2m doubles) x 32 columns x 2 halves x ncols/64 groups; a box = 8 complex K of the
  // 32 columns of one half in two consecutive groups (64 rows of 128 B, swizzled as the 2D box)
  CUtensorMap mapA;
  {
    const cuuint64_t gdim[4] = {(cuuint64_t)(2 * m), 32u, 2u, (cuuint64_t)(ncols / 64)};
    const cuuint64_t gstr[3] = {(cuuint64_t)lda * sizeof(double2),
                                (cuuint64_t)32 * lda * sizeof(double2),
                                (cuuint64_t)64 * lda * sizeof(double2)};
    const cuuint32_t box[4] = {16u, 32u, 1u, 2u};
    const cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
    if (encode(&mapA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)A, gdim, gstr, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  // rows of every product: 48-row tiles, the remainder r = 24 / 32 / 40 on r-row tiles beside
  // them on the aux stream (as sketch_gemm's row split); other remainders pad the last 48-row tile;
  // fewer than 48 rows (C2: 40) on one tile of the smallest height that holds them
  const int h = strassen_main_rows(lh);
  const int rem = lh % 48;
  // (padding the last 48-row tile instead, RID_STR_PAD=1: C4 99.8 vs 91.0 ms, C5 208.2 vs 201.6)
  bool split = aux && aux->stream && lh > 48 && (rem == 24 || rem == 32 || rem == 40);
  if (const char* v = experiment_env("RID_STR_PAD")) split = split && atoi(v) == 0;
  const int main_end = split ? lh - rem : lh;
  if (split) {
    if ((e = cudaEventRecord(aux->fork, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(aux->stream, aux->fork, 0)) != cudaSuccess) return e;
  }
  if ((e = products_rows(h, rem, mapA, Rc, ldc, Rs, lds, M, lh, nh, mh, 0, main_end, st, S)) !=
      cudaSuccess)
    return e;
  *launches += 2;
  if (split) {
    if ((e = products_rows(rem, rem, mapA, Rc, ldc, Rs, lds, M, lh, nh, mh, main_end, lh,
                           aux->stream, S)) != cudaSuccess)
      return e;
    *launches += 2;
    if ((e = cudaEventRecord(aux->join, aux->stream)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st, aux->join, 0)) != cudaSuccess) return e;
  }
  const int64_t total = (int64_t)lh * nh;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_strassen_combine<<<(unsigned)blocks, 256, 0, st>>>(M, lh, nh, S, Y, ldy);
  *launches += 1;
  return cudaGetLastError();
}

}  // namespace rid

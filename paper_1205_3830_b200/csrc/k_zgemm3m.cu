// k_zgemm3m.cu — the sketch Y = R · A (north_star) as three real products on the
// FP64 tensor pipe (DMMA), Gauss's complex multiplication:
//     P1 = Re R · Re A,   P2 = Im R · Im A,   P3 = (Re R + Im R) · (Re A + Im A),
//     Re Y = P1 − P2,     Im Y = P3 − P1 − P2,
// i.e. 6·l·m·n real flops instead of the 8·l·m·n of the real embedding (k_zgemm.cu), a quarter of
// the tensor work of the metric's kernel. Each P is one ascending fma chain over the complex K
// index inside a K slice (DMMA.8x8x4 is that chain, profiles/r01_box_facts_*.txt); Y agrees with
// the oracle's 4-multiplication ascending chain (docs/RNG.md §6) to rounding — reading R31 in
// DESIGN.md (north-star bar 1e-12 relative; the ordered 4M kernel stays selectable with
// RID_SKETCH_4M=1 and is bit-exact).
//
// Fragments (mma.m8n8k4.row.col.f64): M = column j of A (8), N = complex row r of R (8), K =
// complex index i (4 per DMMA). Lane (g, t) = (lane >> 2, lane & 3) loads ONE complex A(i0 + t, j)
// and ONE complex R(r0 + g, i0 + t) per k-step (LDS.128 each) and forms the three fragments
// (re, im, re + im) in registers — half the shared-memory loads of the real embedding per flop.
// Its accumulator pair is (P(j, r0 + 2t), P(j, r0 + 2t + 1)) for each of P1, P2, P3.
// Pipeline as k_zgemm.cu: STAGES-deep cp.async ring; A pitch PB ≡ 8 (mod 16) doubles and R pitch
// PR ≡ 2 (mod 8) complex make every LDS.128 fragment load conflict-free; grid = (row tiles,
// column tiles, K slices) with rows fastest (the CTAs sharing an A tile run together).
#include <cstdlib>

#include "rid_device.cuh"
#include "rid_internal.h"

namespace rid {

template <int FJ, int FR, int WJ, int WR, int BKC, int STAGES, int RS>
struct Z3Cfg {
  static constexpr int kThreads = WJ * WR * 32;
  static constexpr int BJ = WJ * FJ * 8;    // columns per CTA
  static constexpr int BR = WR * FR * 8;    // complex rows per CTA
  static constexpr int PB = 2 * BKC + 8;    // doubles per A column; ≡ 8 (mod 16)
  static constexpr int PR = BR + ((2 - BR % 8) % 8 + 8) % 8;  // complex; ≡ 2 (mod 8)
  static constexpr int PS = BR + ((4 - BR % 16) % 16 + 16) % 16;  // doubles; ≡ 4 (mod 16)
  static constexpr int kStageB = BJ * PB;        // doubles
  static constexpr int kStageR = BKC * PR * 2;   // doubles
  static constexpr int kStageS = RS ? BKC * PS : 0;  // doubles: Re R + Im R (RS = 1)
  static constexpr int kStage = kStageB + kStageR + kStageS;
  static constexpr size_t kSmem = (size_t)STAGES * kStage * sizeof(double);
  static_assert(BKC % 4 == 0, "BKC must be a multiple of 4");
  static_assert(PB % 16 == 8 && PR % 8 == 2 && PR >= BR && PS % 16 == 4 && PS >= BR, "pitches");
  static_assert(BR % 2 == 0, "rows in pairs");
};

// RS = 1: Re R + Im R comes from a precomputed plane (no add per R fragment, 6 KB more shared
// memory per stage); RS = 0: it is formed in registers like the A side. DBUF = 1: the fragments
// of k-step kk + 1 are loaded while the DMMAs of kk issue.
template <int FJ, int FR, int WJ, int WR, int BKC, int STAGES, int MINB, int RS, int DBUF>
__global__ void __launch_bounds__(WJ* WR * 32, MINB)
    k_zgemm3m(const double2* __restrict__ Rm, int64_t ldr, const double* __restrict__ Rs,
              int64_t ldrs, const double2* __restrict__ Bm, int64_t ldb, double2* __restrict__ C,
              int64_t ldc, int64_t Mout, int64_t N, int64_t K, int64_t kchunk, int64_t zstride,
              const Z3Batch bt) {
  using Cfg = Z3Cfg<FJ, FR, WJ, WR, BKC, STAGES, RS>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wj = warp % WJ, wr = warp / WJ;
  const int64_t r0 = (int64_t)blockIdx.x * Cfg::BR;
  const int64_t j0 = (int64_t)blockIdx.y * Cfg::BJ;
  int64_t kbeg = 0;
  if (bt.n > 0) {  // batched: blockIdx.z selects one of bt.n independent products (no K split)
    const int z = blockIdx.z;
    Rm += bt.roff[z];
    Bm += bt.boff[z];
    C += bt.coff[z];
    Mout = bt.mout[z];
    if (r0 >= Mout) return;
  } else {
    kbeg = (int64_t)blockIdx.z * kchunk;
    K = (kbeg + kchunk < K) ? kbeg + kchunk : K;  // end of this K slice
    C += (int64_t)blockIdx.z * zstride;
  }
  const int64_t nk = (K - kbeg + BKC - 1) / BKC;

  // per-thread copy plan, fixed for the K loop (only the K offset moves from stage to stage)
  constexpr int kChB = (Cfg::BJ * BKC + Cfg::kThreads - 1) / Cfg::kThreads;
  constexpr int kChR = (BKC * Cfg::BR + Cfg::kThreads - 1) / Cfg::kThreads;
  constexpr int kChS = RS ? (BKC * Cfg::BR / 2 + Cfg::kThreads - 1) / Cfg::kThreads : 0;
  const double2* srcB[kChB];
  int dstB[kChB], kcB[kChB];
  bool okB[kChB];
#pragma unroll
  for (int i = 0; i < kChB; ++i) {
    const int q = tid + i * Cfg::kThreads;
    const int col = q / BKC, kc = q % BKC;
    okB[i] = q < Cfg::BJ * BKC && j0 + col < N;
    srcB[i] = okB[i] ? Bm + (j0 + col) * ldb + kc : Bm;
    dstB[i] = col * Cfg::PB + 2 * kc;
    kcB[i] = q < Cfg::BJ * BKC ? kc : 0;
  }
  const double2* srcR[kChR];
  int dstR[kChR], kcR[kChR];
  bool okR[kChR], inR[kChR];
#pragma unroll
  for (int i = 0; i < kChR; ++i) {
    const int q = tid + i * Cfg::kThreads;
    const int kc = q / Cfg::BR, rr = q % Cfg::BR;
    inR[i] = q < BKC * Cfg::BR;
    okR[i] = inR[i] && r0 + rr < Mout;
    srcR[i] = okR[i] ? Rm + kc * ldr + r0 + rr : Rm;
    dstR[i] = 2 * (kc * Cfg::PR + rr);
    kcR[i] = inR[i] ? kc : 0;
  }
  // Re R + Im R plane (RS = 1; ldrs even, pad rows zero): pairs of rows per 16-byte chunk
  const double* srcS[kChS > 0 ? kChS : 1];
  int dstS[kChS > 0 ? kChS : 1], kcS[kChS > 0 ? kChS : 1];
  bool okS[kChS > 0 ? kChS : 1], inS[kChS > 0 ? kChS : 1];
#pragma unroll
  for (int i = 0; i < kChS; ++i) {
    const int q = tid + i * Cfg::kThreads;
    const int kc = q / (Cfg::BR / 2), rr = 2 * (q % (Cfg::BR / 2));
    inS[i] = q < BKC * Cfg::BR / 2;
    okS[i] = inS[i] && r0 + rr < Mout;
    srcS[i] = okS[i] ? Rs + kc * ldrs + r0 + rr : Rs;
    dstS[i] = kc * Cfg::PS + rr;
    kcS[i] = inS[i] ? kc : 0;
  }
  auto load_stage = [&](int slot, int64_t kc0) {
    double* sB = smem + (size_t)slot * Cfg::kStage;
    double* sR = sB + Cfg::kStageB;
    double* sS = sR + Cfg::kStageR;
    const bool full = kc0 + BKC <= K;
#pragma unroll
    for (int i = 0; i < kChB; ++i)
      if (tid + i * Cfg::kThreads < Cfg::BJ * BKC) {
        const bool ok = okB[i] && (full || kc0 + kcB[i] < K);
        cp_async16(sB + dstB[i], ok ? srcB[i] + kc0 : Bm, ok);
      }
    const int64_t roff = kc0 * ldr;
#pragma unroll
    for (int i = 0; i < kChR; ++i)
      if (inR[i]) {
        const bool ok = okR[i] && (full || kc0 + kcR[i] < K);
        cp_async16(sR + dstR[i], ok ? srcR[i] + roff : Rm, ok);
      }
    const int64_t soff = kc0 * ldrs;
#pragma unroll
    for (int i = 0; i < kChS; ++i)
      if (inS[i]) {
        const bool ok = okS[i] && (full || kc0 + kcS[i] < K);
        cp_async16(sS + dstS[i], ok ? srcS[i] + soff : Rs, ok);
      }
  };

  double acc[FJ][FR][3][2];
#pragma unroll
  for (int a = 0; a < FJ; ++a)
#pragma unroll
    for (int b = 0; b < FR; ++b)
#pragma unroll
      for (int p = 0; p < 3; ++p) acc[a][b][p][0] = acc[a][b][p][1] = 0.0;

  const int laneB = (wj * FJ * 8 + g) * Cfg::PB + 2 * t;        // doubles: A(i0 + t, j)
  const int laneR = 2 * (t * Cfg::PR + wr * FR * 8 + g);        // doubles: R(r0 + g, i0 + t)
  const int laneS = t * Cfg::PS + wr * FR * 8 + g;              // doubles: Rs(r0 + g, i0 + t)

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, kbeg + (int64_t)s * BKC);
    cp_async_commit();
  }
  for (int64_t kt = 0; kt < nk; ++kt) {
    {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int64_t kn = kt + STAGES - 1;
      if (kn < nk) load_stage((int)(kn % STAGES), kbeg + kn * BKC);
      cp_async_commit();
    }
    const double* sB = smem + (size_t)(kt % STAGES) * Cfg::kStage;
    const double* sR = sB + Cfg::kStageB;
    const double* sS = sR + Cfg::kStageR;
    double a[DBUF + 1][FJ][3], b[DBUF + 1][FR][3];
    auto frag = [&](int kk, int buf) {
#pragma unroll
      for (int f = 0; f < FJ; ++f) {
        const double2 v = *reinterpret_cast<const double2*>(sB + laneB + f * 8 * Cfg::PB + kk * 8);
        a[buf][f][0] = v.x;
        a[buf][f][1] = v.y;
        a[buf][f][2] = __dadd_rn(v.x, v.y);  // FP64 pipe, shared with DMMA
      }
#pragma unroll
      for (int f = 0; f < FR; ++f) {
        const double2 v = *reinterpret_cast<const double2*>(sR + laneR + f * 16 + kk * 8 * Cfg::PR);
        b[buf][f][0] = v.x;
        b[buf][f][1] = v.y;
        b[buf][f][2] = RS ? sS[laneS + f * 8 + kk * 4 * Cfg::PS] : __dadd_rn(v.x, v.y);
      }
    };
    if (DBUF) frag(0, 0);
#pragma unroll
    for (int kk = 0; kk < BKC / 4; ++kk) {
      const int cur = DBUF ? (kk & 1) : 0;
      if (DBUF) {
        if (kk + 1 < BKC / 4) frag(kk + 1, (kk + 1) & 1);
      } else {
        frag(kk, 0);
      }
#pragma unroll
      for (int fa = 0; fa < FJ; ++fa)
#pragma unroll
        for (int fb = 0; fb < FR; ++fb)
#pragma unroll
          for (int p = 0; p < 3; ++p)
            dmma8x8x4(acc[fa][fb][p][0], acc[fa][fb][p][1], a[cur][fa][p], b[cur][fb][p]);
    }
  }
  cp_async_wait<0>();

  // epilogue: lane (g, t) holds rows r0 + wr*FR*8 + fb*8 + 2t + {0, 1} of column j0 + ... + g
#pragma unroll
  for (int fa = 0; fa < FJ; ++fa) {
    const int64_t j = j0 + wj * FJ * 8 + fa * 8 + g;
    if (j >= N) continue;
#pragma unroll
    for (int fb = 0; fb < FR; ++fb) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = r0 + wr * FR * 8 + fb * 8 + 2 * t + h;
        if (r >= Mout) continue;
        const double p1 = acc[fa][fb][0][h], p2 = acc[fa][fb][1][h], p3 = acc[fa][fb][2][h];
        C[j * ldc + r] = make_double2(__dsub_rn(p1, p2), __dsub_rn(__dsub_rn(p3, p1), p2));
      }
    }
  }
}

__global__ void k_splitk_reduce3(const double2* __restrict__ part, int S, int64_t Mout, int64_t N,
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

template <int FJ, int FR, int WJ, int WR, int BKC, int STAGES, int MINB, int RS, int DBUF>
static cudaError_t launch3(const double2* Rm, int64_t ldr, const double* Rs, int64_t ldrs,
                           const double2* Bm, int64_t ldb, double2* C, int64_t ldc, int64_t Mout,
                           int64_t N, int64_t K, cudaStream_t st, int S, double2* partial) {
  using Cfg = Z3Cfg<FJ, FR, WJ, WR, BKC, STAGES, RS>;
  auto kern = k_zgemm3m<FJ, FR, WJ, WR, BKC, STAGES, MINB, RS, DBUF>;
  {
    const cudaError_t e = ensure_dyn_smem((const void*)kern, Cfg::kSmem);
    if (e != cudaSuccess) return e;
  }
  const int64_t tiles_r = (Mout + Cfg::BR - 1) / Cfg::BR;
  const int64_t tiles_j = (N + Cfg::BJ - 1) / Cfg::BJ;
  int64_t kc = K > 0 ? K : 1;
  double2* Cout = C;
  int64_t ldo = ldc, zs = 0;
  if (S > 1 && partial) {
    kc = (K + S - 1) / S;
    kc = ((kc + BKC - 1) / BKC) * BKC;
    S = (int)((K + kc - 1) / kc);
    if (S > 1) {
      Cout = partial;
      ldo = Mout;
      zs = Mout * N;
    }
  } else {
    S = 1;
  }
  if (tiles_r > 0x7FFFFFFF || tiles_j > 65535 || S > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)tiles_r, (unsigned)tiles_j, (unsigned)S);
  Z3Batch none{};
  kern<<<grid, Cfg::kThreads, Cfg::kSmem, st>>>(Rm, ldr, Rs, ldrs, Bm, ldb, Cout, ldo, Mout, N, K,
                                                kc, zs, none);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || S == 1) return e;
  int64_t blocks = (Mout * N + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_splitk_reduce3<<<(unsigned)blocks, 256, 0, st>>>(partial, S, Mout, N, C, ldc);
  return cudaGetLastError();
}

template <int FJ, int FR, int WJ, int WR, int BKC, int STAGES, int MINB>
static cudaError_t launch3_batched(const double2* Rm, int64_t ldr, const double2* Bm, int64_t ldb,
                                   double2* C, int64_t ldc, const Z3Batch& bt, int64_t N, int64_t K,
                                   cudaStream_t st) {
  using Cfg = Z3Cfg<FJ, FR, WJ, WR, BKC, STAGES, 0>;
  auto kern = k_zgemm3m<FJ, FR, WJ, WR, BKC, STAGES, MINB, 0, 0>;
  {
    const cudaError_t e = ensure_dyn_smem((const void*)kern, Cfg::kSmem);
    if (e != cudaSuccess) return e;
  }
  int64_t mmax = 0;
  for (int z = 0; z < bt.n; ++z) mmax = bt.mout[z] > mmax ? bt.mout[z] : mmax;
  const int64_t tiles_r = (mmax + Cfg::BR - 1) / Cfg::BR;
  const int64_t tiles_j = (N + Cfg::BJ - 1) / Cfg::BJ;
  if (tiles_r < 1 || tiles_j > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)tiles_r, (unsigned)tiles_j, (unsigned)bt.n);
  kern<<<grid, Cfg::kThreads, Cfg::kSmem, st>>>(Rm, ldr, nullptr, 0, Bm, ldb, C, ldc, mmax, N, K, K,
                                                0, bt);
  return cudaGetLastError();
}

// Tile candidates (complex rows per CTA x columns): every row of l is real work, so the one that
// pads the fewest rows wins (ties -> more rows per tile: fewer re-reads of A). 8 warps, 2 CTAs
// per SM, 16 complex K per stage (tools/tune_3m.py, measured on B200):
//   id 0: 48 rows (2 x 3 fragments) x 64 columns, R sums in registers   C3 (144), C4 (528)
//         C4: 108.7 ms = 41.7 TF/s in the 8lmn convention (31.3 TF/s executed, 84% of DMMA peak)
//   id 1: 40 rows (1 x 5) x 64 columns, precomputed R sums, fragments double-buffered
//         C5 (272 -> 280): 232 ms = 40.2 TF/s (30.2 executed); C2 (80)
//   id 2: 24 rows (1 x 3) x 64 columns, as id 1                          C1 (24)
static int pick3(int64_t Mout) {
  const int rows[3] = {48, 40, 24};
  if (const char* v = experiment_env("RID_Z3_ROWS")) {  // tile-height experiments (tools/tma_sketch_time.py)
    for (int i = 0; i < 3; ++i)
      if (atoi(v) == rows[i]) return i;
  }
  int best = 0;
  int64_t bw = INT64_MAX, br = 0;
  for (int i = 0; i < 3; ++i) {
    const int64_t w = ((Mout + rows[i] - 1) / rows[i]) * rows[i] - Mout;
    if (w < bw || (w == bw && rows[i] > br)) {
      bw = w;
      br = rows[i];
      best = i;
    }
  }
  return best;
}
static int rows3(int id) {
  const int rows[3] = {48, 40, 24};
  return rows[id];
}
int zgemm3m_tile_rows(int64_t Mout) { return rows3(pick3(Mout)); }

int zgemm3m_ksplit(int64_t Mout, int64_t K, int64_t n_ref, int num_sms) {
  if (const char* v = select_env("RID_SKETCH_SPLIT")) {
    const int s = atoi(v);
    if (s >= 1) return s;
  }
  if (n_ref <= 0 || K <= 0) return 1;
  const int64_t tiles = ((n_ref + 63) / 64) * ((Mout + rows3(pick3(Mout)) - 1) / rows3(pick3(Mout)));
  int64_t s = (2 * (int64_t)num_sms + tiles - 1) / tiles;
  // slices of at least 128 complex K (8 stages): binds only when the tiles are very few (C1:
  // 8 slices, sketch 30 -> ~8 us); the larger configs' slice counts come from the tile count
  const int64_t smax = K / 128 > 1 ? K / 128 : 1;
  if (s > smax) s = smax;
  if (s > 64) s = 64;
  return s < 1 ? 1 : (int)s;
}

// Rs(r, i) = Re R(r, i) + Im R(r, i), ldrs = l rounded up to even, pad rows zero
__global__ void k_rsum(const double2* __restrict__ R, int64_t l, int64_t m, int64_t ldr,
                       double* __restrict__ Rs, int64_t ldrs) {
  const int64_t total = ldrs * m;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / ldrs, r = q % ldrs;
    double v = 0.0;
    if (r < l) {
      const double2 x = R[i * ldr + r];
      v = __dadd_rn(x.x, x.y);
    }
    Rs[q] = v;
  }
}

cudaError_t rsum_fill(const double2* R, int64_t l, int64_t m, int64_t ldr, double* Rs,
                      int64_t ldrs, cudaStream_t st) {
  if (l <= 0 || m <= 0) return cudaSuccess;
  int64_t blocks = (ldrs * m + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_rsum<<<(unsigned)blocks, 256, 0, st>>>(R, l, m, ldr, Rs, ldrs);
  return cudaGetLastError();
}

cudaError_t zgemm3m(const double2* Rm, int64_t ldr, const double* Rs, int64_t ldrs,
                    const double2* Bm, int64_t ldb, double2* C, int64_t ldc, int64_t Mout,
                    int64_t N, int64_t K, cudaStream_t st, int ksplit, double2* partial) {
  if (Mout <= 0 || N <= 0) return cudaSuccess;
#define RID_L3(...) launch3<__VA_ARGS__>(Rm, ldr, Rs, ldrs, Bm, ldb, C, ldc, Mout, N, K, st, ksplit, partial)
  if (const char* v = experiment_env("RID_Z3_VARIANT")) {  // tile experiments (tools/sketch3m_check.py)
    switch (atoi(v)) {
      case 1: return RID_L3(2, 3, 4, 2, 16, 3, 2, 0, 0);
      case 2: return RID_L3(2, 3, 4, 2, 16, 3, 2, 0, 1);
      case 3: return RID_L3(2, 3, 4, 2, 16, 3, 2, 1, 0);
      case 4: return RID_L3(2, 3, 4, 2, 8, 4, 2, 1, 1);
      case 5: return RID_L3(1, 5, 8, 1, 16, 3, 2, 0, 0);
      case 6: return RID_L3(1, 5, 8, 1, 16, 3, 2, 1, 1);
      case 7: return RID_L3(1, 5, 8, 1, 16, 3, 2, 0, 1);
      case 8: return RID_L3(1, 6, 8, 1, 16, 3, 2, 0, 0);
      case 9: return RID_L3(1, 6, 8, 1, 16, 3, 2, 1, 1);
      case 10: return RID_L3(2, 3, 4, 2, 8, 4, 2, 0, 0);
      case 11: return RID_L3(1, 3, 8, 1, 16, 3, 2, 1, 1);
      default: break;
    }
  }
  if (zgemm3m_tma_enabled(Mout))
    return zgemm3m_tma(Rm, ldr, Rs, ldrs, Bm, ldb, C, ldc, Mout, N, K, st, ksplit, partial);
  if (!Rs) {  // no Re R + Im R plane (e.g. the SRFT's row-grouped W): sums in registers
    switch (pick3(Mout)) {
      case 0: return RID_L3(2, 3, 4, 2, 16, 3, 2, 0, 0);
      case 1: return RID_L3(1, 5, 8, 1, 16, 3, 2, 0, 0);
      default: return RID_L3(1, 3, 8, 1, 16, 3, 2, 0, 0);
    }
  }
  switch (pick3(Mout)) {
    case 0: return RID_L3(2, 3, 4, 2, 16, 3, 2, 0, 0);
    case 1: return RID_L3(1, 5, 8, 1, 16, 3, 2, 1, 1);
    default: return RID_L3(1, 3, 8, 1, 16, 3, 2, 1, 1);
  }
#undef RID_L3
}

cudaError_t zgemm3m_batched(const double2* Rm, int64_t ldr, const double2* Bm, int64_t ldb,
                            double2* C, int64_t ldc, const Z3Batch& bt, int64_t N, int64_t K,
                            cudaStream_t st) {
  if (bt.n <= 0 || N <= 0) return cudaSuccess;
  if (bt.n > kZ3BatchMax) return cudaErrorInvalidValue;
  int64_t mmax = 0;
  for (int z = 0; z < bt.n; ++z) mmax = bt.mout[z] > mmax ? bt.mout[z] : mmax;
  switch (pick3(mmax)) {
    case 0: return launch3_batched<2, 3, 4, 2, 16, 3, 2>(Rm, ldr, Bm, ldb, C, ldc, bt, N, K, st);
    case 1: return launch3_batched<1, 5, 8, 1, 16, 3, 2>(Rm, ldr, Bm, ldb, C, ldc, bt, N, K, st);
    default: return launch3_batched<1, 3, 8, 1, 16, 3, 2>(Rm, ldr, Bm, ldb, C, ldc, bt, N, K, st);
  }
}

int sketch_mults() {
  const char* v = select_env("RID_SKETCH_4M");
  return (v && atoi(v) != 0) ? 4 : 3;
}
int sketch_ksplit(int64_t l, int64_t m, int64_t n_ref, int num_sms) {
  return sketch_mults() == 4 ? zgemm_ksplit(l, m, n_ref, num_sms)
                             : zgemm3m_ksplit(l, m, n_ref, num_sms);
}
// Wave quantisation of the unsplit sketch: R_t row tiles x T column tiles over 2 CTAs per SM.
// When the last wave would run only a few CTAs (C4: 5632 = 19 x 296 + 8), the trailing global
// column tiles that fall into it are computed with a K split instead, sized to fill one wave
// (C4: the last 64 columns in 26 slices). The set depends only on (l, m, n) and the SM count, so
// every column of Y is still bitwise independent of the sharding.
SketchTail sketch_tail(int64_t l, int64_t m, int64_t n, int num_sms) {
  SketchTail t{0, 1};
  if (sketch_mults() != 3 || select_env("RID_SKETCH_SPLIT") || select_env("RID_SKETCH_NOTAIL")) return t;
  if (zgemm3m_ksplit(l, m, n / 8, num_sms) != 1) return t;  // already split everywhere
  const int64_t rt = (l + rows3(pick3(l)) - 1) / rows3(pick3(l));
  const int64_t T = (n + 63) / 64, slots = 2 * (int64_t)num_sms, total = rt * T;
  const int64_t rem = total % slots;
  if (rem == 0 || rem * 2 >= slots) return t;
  const int64_t q = (rem + rt - 1) / rt;  // trailing column tiles in the split set
  if (q >= T) return t;
  int64_t S = slots / (q * rt);
  const int64_t smax = m / 512 > 1 ? m / 512 : 1;
  if (S > smax) S = smax;
  if (S > 64) S = 64;
  if (S < 2) return t;
  t.cols = n - (T - q) * 64;
  t.S = (int)S;
  return t;
}

int64_t sketch_partial_elems(int64_t l, int64_t m, int64_t n, int64_t ncols, int num_sms) {
  const int S = sketch_ksplit(l, m, n / 8, num_sms);
  const SketchTail t = sketch_tail(l, m, n, num_sms);
  const int64_t a = S > 1 ? (int64_t)S * l * ncols : 0;
  const int64_t b = t.cols > 0 ? (int64_t)t.S * l * (t.cols < ncols ? t.cols : ncols) : 0;
  return a > b ? a : b;
}

cudaError_t sketch_gemm(const double2* R, int64_t ldr, const double* Rs, const double2* A,
                        int64_t lda, double2* Y, int64_t ldy, int64_t l, int64_t ncols, int64_t m,
                        cudaStream_t st, int ksplit, double2* partial, int64_t col0, int64_t n,
                        int num_sms, int* launches, const SketchAux* aux) {
  int dummy = 0;
  if (!launches) launches = &dummy;
  if (sketch_mults() == 4) {
    *launches += ksplit > 1 ? 2 : 1;
    return zgemm_ordered(R, ldr, A, lda, Y, ldy, l, ncols, m, 0, 0.0, 0, 0, st, ksplit, partial);
  }
  const SketchTail t = (ksplit == 1 && partial) ? sketch_tail(l, m, n, num_sms) : SketchTail{0, 1};
  const int64_t tail0 = n - t.cols;  // first global column of the split set
  int64_t nmain = ncols;
  if (t.cols > 0 && col0 + ncols > tail0) nmain = tail0 > col0 ? tail0 - col0 : 0;
  cudaError_t e = cudaSuccess;
  // row split: when the 48-row tile (the most efficient) does not divide l but l = 48 a + r with
  // r a tile height of its own (24 / 32 / 40, e.g. C5: 272 = 5 x 48 + 32), rows [0, 48 a) run on
  // 48-row tiles and the last r rows on r-row tiles (aux stream) instead of padding l to a single
  // height (C5: 40-row tiles, 280 rows). Each element's chain is the same: Y is bitwise unchanged.
  // (only with the aux stream: run serially after the main part, the r-row part's lone partial
  // wave costs more than the padding saves, e.g. the e2e path's 1 GiB column chunks)
  int rsplit = 0;
  if (aux && aux->stream && zgemm3m_tma_enabled(l) && Rs && l > 48 &&
      !select_env("RID_SKETCH_NOROWSPLIT")) {
    const int64_t r = l % 48;
    if (r == 24 || r == 32 || r == 40) rsplit = (int)r;
  }
  const bool use_aux = aux && aux->stream;
  // the K-split tail set (and the r-row part) run on the aux stream, launched after the main
  // product so their CTAs take the SMs the main launch's last wave leaves idle
  const bool fork = use_aux && nmain > 0 && (nmain < ncols || rsplit);
  if (fork) {
    if ((e = cudaEventRecord(aux->fork, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(aux->stream, aux->fork, 0)) != cudaSuccess) return e;
  }
  if (nmain > 0 && rsplit) {
    const int64_t l48 = l - rsplit;
    e = zgemm3m_tma_rows(R, ldr, Rs, rsum_ld(l), A, lda, Y, ldy, l48, nmain, m, st, ksplit,
                         partial, 48);
    *launches += ksplit > 1 ? 2 : 1;
    if (e != cudaSuccess) return e;
    e = zgemm3m_tma_rows(R + l48, ldr, Rs + l48, rsum_ld(l), A, lda, Y + l48, ldy, rsplit, nmain,
                         m, fork ? aux->stream : st, ksplit,
                         partial ? partial + (int64_t)ksplit * l48 * nmain : nullptr, rsplit);
    *launches += ksplit > 1 ? 2 : 1;
    if (e != cudaSuccess) return e;
  } else if (nmain > 0) {
    e = zgemm3m(R, ldr, Rs, rsum_ld(l), A, lda, Y, ldy, l, nmain, m, st, ksplit, partial);
    *launches += ksplit > 1 ? 2 : 1;
    if (e != cudaSuccess) return e;
  }
  if (nmain < ncols) {
    // (the tail's partials may not overlap the r-row part's, which runs concurrently)
    double2* tpart = partial;
    if (fork && rsplit && ksplit > 1) tpart = nullptr;  // not reached: the tail set needs S = 1
    e = zgemm3m(R, ldr, Rs, rsum_ld(l), A + nmain * lda, lda, Y + nmain * ldy, ldy, l,
                ncols - nmain, m, fork ? aux->stream : st, t.S, tpart);
    *launches += 2;
    if (e != cudaSuccess) return e;
  }
  if (fork) {
    if ((e = cudaEventRecord(aux->join, aux->stream)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st, aux->join, 0)) != cudaSuccess) return e;
  }
  return e;
}

}  // namespace rid

// k_zgemm.cu — the ordered complex128 GEMM on the FP64 tensor pipe (DMMA), used by three steps:
//   * rid_sketch:    Y  = R · A          (Mout = l,  K = m, N = n_loc)   north_star
//   * rid_generate:  A  = X · Y0 + ε·E   (Mout = m,  K = k, N = n_loc)   PAPER.md:112; RNG.md §5
//   * interpolation: T  = R11⁻¹ · R12    (Mout = k,  K = k, N = n_loc)   PAPER.md:88-90 (Eq. 10)
//
// Real embedding: a complex product C = Rm·Bm is computed as C̃ᵀ = B̃ᵀ · R̃ᵀ where B̃ is Bm's
// interleaved (re, im) memory read as a 2K × N real matrix (no copy) and R̃ is the 2×2-block
// expansion [[re, −im], [im, re]] of Rm built on the fly from Rm's own bits. The MMA's M dimension
// is the column index j, its N dimension the real row index r̃ = 2r + {re, im}, so each lane's
// accumulator pair {c0, c1} is exactly one complex output (re, im) — stored as one 16-byte write.
//
// Order: every output element is ONE fused-multiply-add chain over the real K index in ascending
// order (DMMA.8x8x4 is that chain, bit for bit — measured, profiles/r01_box_facts_*.txt), starting
// from +0. For the sketch and the generation this is exactly the order of docs/RNG.md §5/§6, so
// the results are bit-identical to the oracle's naive loops. No split-K: the K loop is sequential.
//
// Pipeline: STAGES-deep cp.async (LDGSTS) ring into padded shared memory (B̃ pitch ≡ 4 mod 16
// doubles and R pitch ≡ 4 mod 8 complex make every fragment load a single conflict-free
// wavefront); 8 warps; grid = (r̃-tiles, j-tiles) with r̃ fastest so the CTAs that share an
// A tile run together and hit L2.
#include <cstdlib>

#include "rid_device.cuh"
#include "rid_internal.h"

namespace rid {

struct ZgemmEpilogue {
  int mode;          // 0: C = acc; 1: C = fma(noise, E(i, col0 + j), acc) (generation);
                     // 2: C = C - acc (QRCP trailing update)
  double noise;
  uint64_t seed;
  int64_t col0;
  int64_t kchunk;    // complex K per blockIdx.z slice (K when there is no split)
  int64_t zstride;   // elements between the partial outputs of consecutive slices
  int regen_stream;  // REGEN kernels: Philox stream of R
};

template <int FJ, int FR, int WARPS_J, int WARPS_R, int BK, int STAGES>
struct ZgemmCfg {
  static constexpr int kThreads = WARPS_J * WARPS_R * 32;
  static constexpr int BJ = WARPS_J * FJ * 8;   // columns per CTA
  static constexpr int BR = WARPS_R * FR * 8;   // real rows per CTA
  static constexpr int BRC = BR / 2;            // complex rows per CTA
  static constexpr int BKC = BK / 2;            // complex K per stage
  static constexpr int PB = BK + 4;             // doubles; ≡ 4 (mod 16)
  static constexpr int PR = BRC + ((4 - BRC % 8) % 8 + 8) % 8;  // complex; ≡ 4 (mod 8)
  static constexpr int kStageB = BJ * PB;        // doubles
  static constexpr int kStageR = BKC * PR * 2;   // doubles
  static constexpr int kStage = kStageB + kStageR;
  static constexpr size_t kSmem = (size_t)STAGES * kStage * sizeof(double);
  static_assert(BK % 16 == 0, "BK must be a multiple of 16");
  static_assert(PR % 8 == 4 && PR >= BRC, "R pitch");
};

// REGEN = 1: the R tile is regenerated from Philox inside the kernel (R(r, i) = N(seed,
// ep.regen_stream, r, i), the north star's literal design) instead of streamed from the
// pre-generated R in HBM/L2 — kept as the measured alternative.
template <int FJ, int FR, int WARPS_J, int WARPS_R, int BK, int STAGES, int MINB, int REGEN = 0>
__global__ void __launch_bounds__(WARPS_J* WARPS_R * 32, MINB)
    k_zgemm_dmma(const double2* __restrict__ Rm, int64_t ldr, const double2* __restrict__ Bm,
                 int64_t ldb, double2* __restrict__ C, int64_t ldc, int64_t Mout, int64_t N,
                 int64_t K, ZgemmEpilogue ep) {
  using Cfg = ZgemmCfg<FJ, FR, WARPS_J, WARPS_R, BK, STAGES>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wj = warp % WARPS_J, wr = warp / WARPS_J;
  const int64_t r0c = (int64_t)blockIdx.x * Cfg::BRC;  // complex row offset of this CTA
  const int64_t j0 = (int64_t)blockIdx.y * Cfg::BJ;
  // K slice of this CTA (split-K: blockIdx.z; the slice's partial goes to its own output)
  const int64_t kbeg = (int64_t)blockIdx.z * ep.kchunk;
  K = (kbeg + ep.kchunk < K) ? kbeg + ep.kchunk : K;   // end of the slice
  C += (int64_t)blockIdx.z * ep.zstride;
  const int64_t nk = (K - kbeg + Cfg::BKC - 1) / Cfg::BKC;  // complex-K stages

  // Per-thread copy plan, fixed for the whole K loop: chunk q of the B̃ tile is (column q / BKC,
  // complex K q % BKC), chunk q of the R tile is (K q / BRC, row q % BRC). Only the K offset
  // changes from stage to stage, so each stage is a handful of 64-bit adds and LDGSTS.
  constexpr int kChB = (Cfg::BJ * Cfg::BKC + Cfg::kThreads - 1) / Cfg::kThreads;
  constexpr int kChR = (Cfg::BKC * Cfg::BRC + Cfg::kThreads - 1) / Cfg::kThreads;
  const double2* srcB[kChB];
  int dstB[kChB], kcB[kChB];
  bool okB[kChB];
#pragma unroll
  for (int i = 0; i < kChB; ++i) {
    const int q = tid + i * Cfg::kThreads;
    const int col = q / Cfg::BKC, kc = q % Cfg::BKC;
    okB[i] = q < Cfg::BJ * Cfg::BKC && j0 + col < N;
    srcB[i] = okB[i] ? Bm + (j0 + col) * ldb + kc : Bm;
    dstB[i] = col * Cfg::PB + 2 * kc;
    kcB[i] = q < Cfg::BJ * Cfg::BKC ? kc : 0;
  }
  const double2* srcR[kChR];
  int dstR[kChR], kcR[kChR];
  bool okR[kChR], inR[kChR];
#pragma unroll
  for (int i = 0; i < kChR; ++i) {
    const int q = tid + i * Cfg::kThreads;
    const int kc = q / Cfg::BRC, rr = q % Cfg::BRC;
    inR[i] = q < Cfg::BKC * Cfg::BRC;
    okR[i] = inR[i] && r0c + rr < Mout;
    srcR[i] = okR[i] ? Rm + kc * ldr + r0c + rr : Rm;
    dstR[i] = 2 * (kc * Cfg::PR + rr);
    kcR[i] = inR[i] ? kc : 0;
  }
  auto load_stage = [&](int slot, int64_t kc0) {
    double* sB = smem + (size_t)slot * Cfg::kStage;
    double* sR = sB + Cfg::kStageB;
    const bool full = kc0 + Cfg::BKC <= K;  // only the last stage has a K tail
#pragma unroll
    for (int i = 0; i < kChB; ++i) {
      if (tid + i * Cfg::kThreads < Cfg::BJ * Cfg::BKC) {
        const bool ok = okB[i] && (full || kc0 + kcB[i] < K);
        cp_async16(sB + dstB[i], ok ? srcB[i] + kc0 : Bm, ok);
      }
    }
    const int64_t roff = kc0 * ldr;
#pragma unroll
    for (int i = 0; i < kChR; ++i) {
      if (inR[i]) {
        const bool ok = okR[i] && (full || kc0 + kcR[i] < K);
        if (REGEN) {
          const int q = tid + i * Cfg::kThreads;
          const int64_t gr = r0c + q % Cfg::BRC, gk = kc0 + kcR[i];
          const double2 v = ok ? rid_normal(ep.seed, (uint32_t)ep.regen_stream, (uint32_t)gr,
                                            (uint32_t)gk)
                               : make_double2(0.0, 0.0);
          *reinterpret_cast<double2*>(sR + dstR[i]) = v;
        } else {
          cp_async16(sR + dstR[i], ok ? srcR[i] + roff : Rm, ok);
        }
      }
    }
  };

  double acc[FJ][FR][2];
#pragma unroll
  for (int a = 0; a < FJ; ++a)
#pragma unroll
    for (int b = 0; b < FR; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // per-lane constants of the R̃ fragment: element R̃[r̃][κ] with r̃ parity = g&1, κ parity = t&1
  const int comp = (g & 1) ^ (t & 1);                 // 0 -> re, 1 -> im
  const unsigned long long sgn = ((g & 1) == 0 && (t & 1) == 1) ? 0x8000000000000000ULL : 0ULL;
  const int laneR = 2 * ((t >> 1) * Cfg::PR + (g >> 1)) + comp + wr * FR * 8;  // doubles
  const int laneB = (wj * FJ * 8 + g) * Cfg::PB + t;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, kbeg + (int64_t)s * Cfg::BKC);
    cp_async_commit();
  }

  for (int64_t kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {  // prefetch stage kt + STAGES - 1 into the slot freed by stage kt - 1
      const int64_t kn = kt + STAGES - 1;
      if (kn < nk) load_stage((int)(kn % STAGES), kbeg + kn * Cfg::BKC);
      cp_async_commit();
    }
    const double* sB = smem + (size_t)(kt % STAGES) * Cfg::kStage;
    const double* sR = sB + Cfg::kStageB;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[FJ], b[FR];
#pragma unroll
      for (int f = 0; f < FJ; ++f) a[f] = sB[laneB + f * 8 * Cfg::PB + kk * 4];
#pragma unroll
      for (int f = 0; f < FR; ++f) {
        const double v = sR[laneR + f * 8 + kk * 4 * Cfg::PR];
        b[f] = __longlong_as_double(__double_as_longlong(v) ^ sgn);
      }
#pragma unroll
      for (int fa = 0; fa < FJ; ++fa)
#pragma unroll
        for (int fb = 0; fb < FR; ++fb) dmma8x8x4(acc[fa][fb][0], acc[fa][fb][1], a[fa], b[fb]);
    }
  }
  cp_async_wait<0>();

  // epilogue: {c0, c1} = (re, im) of C(r, j), r = r0c + wr*FR*4 + f*4 + t, j = j0 + wj*FJ*8 + fa*8 + g
#pragma unroll
  for (int fa = 0; fa < FJ; ++fa) {
    const int64_t j = j0 + wj * FJ * 8 + fa * 8 + g;
    if (j >= N) continue;
#pragma unroll
    for (int fb = 0; fb < FR; ++fb) {
      const int64_t r = r0c + wr * FR * 4 + fb * 4 + t;
      if (r >= Mout) continue;
      double2 o = make_double2(acc[fa][fb][0], acc[fa][fb][1]);
      if (ep.mode == 2) {  // QRCP trailing update: C = C - Rm·Bm
        const double2 c = C[j * ldc + r];
        o = make_double2(__dsub_rn(c.x, o.x), __dsub_rn(c.y, o.y));
      }
      C[j * ldc + r] = o;
    }
  }
  if (ep.mode == 1) {
    // generation: A = fma(noise, E, X·Y0) per component, E(i, j) = N(seed, 3, i, col0 + j).
    // A second, rolled pass over this thread's own outputs (just written, L1/L2-hot) keeps the
    // accumulator registers free of the Philox/normal code.
#pragma unroll 1
    for (int q = 0; q < FJ * FR; ++q) {
      const int fa = q / FR, fb = q % FR;
      const int64_t j = j0 + wj * FJ * 8 + fa * 8 + g;
      const int64_t r = r0c + wr * FR * 4 + fb * 4 + t;
      if (j >= N || r >= Mout) continue;
      double2* cp = C + j * ldc + r;
      const double2 a = *cp;
      const double2 e = rid_normal(ep.seed, 3u, (uint32_t)r, (uint32_t)(ep.col0 + j));
      *cp = make_double2(__fma_rn(ep.noise, e.x, a.x), __fma_rn(ep.noise, e.y, a.y));
    }
  }
}

// Split-K combine: C(r, j) = ((P_0 + P_1) + P_2) + ... in slice order (deterministic).
__global__ void k_splitk_reduce(const double2* __restrict__ part, int S, int64_t Mout, int64_t N,
                                double2* __restrict__ C, int64_t ldc) {
  const int64_t total = Mout * N, zs = Mout * N;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    double2 a = part[q];
    for (int z = 1; z < S; ++z) {
      const double2 b = part[z * zs + q];
      a = make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
    }
    const int64_t r = q % Mout, j = q / Mout;
    C[j * ldc + r] = a;
  }
}

template <int FJ, int FR, int WARPS_J, int WARPS_R, int BK, int STAGES, int MINB = 1, int REGEN = 0>
static cudaError_t launch_cfg(const double2* Rm, int64_t ldr, const double2* Bm, int64_t ldb,
                              double2* C, int64_t ldc, int64_t Mout, int64_t N, int64_t K,
                              const ZgemmEpilogue& ep, cudaStream_t st, int ksplit = 1,
                              double2* partial = nullptr) {
  using Cfg = ZgemmCfg<FJ, FR, WARPS_J, WARPS_R, BK, STAGES>;
  auto kern = k_zgemm_dmma<FJ, FR, WARPS_J, WARPS_R, BK, STAGES, MINB, REGEN>;
  {
    const cudaError_t e = ensure_dyn_smem((const void*)kern, Cfg::kSmem);
    if (e != cudaSuccess) return e;
  }
  const int64_t tiles_r = (Mout + Cfg::BRC - 1) / Cfg::BRC;
  const int64_t tiles_j = (N + Cfg::BJ - 1) / Cfg::BJ;
  ZgemmEpilogue e2 = ep;
  double2* Cout = C;
  int64_t ldo = ldc;
  int S = 1;
  e2.kchunk = K > 0 ? K : 1;
  e2.zstride = 0;
  if (ksplit > 1 && partial && ep.mode == 0) {
    int64_t kc = (K + ksplit - 1) / ksplit;
    kc = ((kc + Cfg::BKC - 1) / Cfg::BKC) * Cfg::BKC;
    S = (int)((K + kc - 1) / kc);
    if (S > 1) {
      e2.kchunk = kc;
      e2.zstride = Mout * N;
      Cout = partial;
      ldo = Mout;
    }
  }
  if (tiles_r > 0x7FFFFFFF || tiles_j > 65535 || S > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)tiles_r, (unsigned)tiles_j, (unsigned)S);
  kern<<<grid, Cfg::kThreads, Cfg::kSmem, st>>>(Rm, ldr, Bm, ldb, Cout, ldo, Mout, N, K, e2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || S == 1) return e;
  int64_t blocks = (Mout * N + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_splitk_reduce<<<(unsigned)blocks, 256, 0, st>>>(partial, S, Mout, N, C, ldc);
  return cudaGetLastError();
}

// Tile choice (tuned on B200, tools/tune_sketch.py / tune_gen.py, profiles/r01_tune_*.log):
// every config runs 3 cp.async stages and 2 CTAs per SM (16 warps/SM hide the DMMA, LDS and
// barrier latencies that 8 warps could not). The 2*Mout real rows are covered by tiles of BR rows;
// the candidate minimising padded rows (every padded row is wasted DMMA work) wins, ties -> the
// larger BR (fewer re-reads of A). FR <= 11: 2 x 4 warps (BJ = 64, BR = 16 FR); FR = 12, 17:
// 8 warps along j (BJ = 64, BR = 8 FR, fits 128 registers). Generation (Mout >= 2048): 64 x 64
// tiles, 3 CTAs per SM. Measured: C4 sketch 34.7 TF/s, C5 33.6, generation C4 30.9.
#define RID_FR_A(X) X(3) X(4) X(5) X(6) X(8) X(9) X(10) X(11)
#define RID_FR_B(X) X(12) X(17)

int zgemm_pick_fr(int64_t Mout) {
  const int64_t rows = 2 * Mout;
  int best = -1;
  int64_t best_waste = INT64_MAX, best_br = 0;
#define RID_TRY(FRV, BRV)                                                        \
  {                                                                              \
    const int64_t br = (BRV);                                                    \
    const int64_t waste = ((rows + br - 1) / br) * br - rows;                    \
    if (waste < best_waste || (waste == best_waste && br > best_br)) {           \
      best_waste = waste;                                                        \
      best_br = br;                                                              \
      best = (FRV);                                                              \
    }                                                                            \
  }
#define RID_TRY_A(FRV) RID_TRY(FRV, 16 * (FRV))
#define RID_TRY_B(FRV) RID_TRY(FRV, 8 * (FRV))
  RID_FR_A(RID_TRY_A)
  RID_FR_B(RID_TRY_B)
#undef RID_TRY_A
#undef RID_TRY_B
#undef RID_TRY
  return best;
}

// Split-K policy for the sketch (K = m long, few output tiles): every rank of a G <= 8 column
// sharding must see enough CTAs, and every column must be computed identically for any G, so the
// slice count depends only on (Mout, K, n_ref) with n_ref = n_global / 8 (the smallest shard an
// 8-GPU box runs): S = ceil(2 * SMs / tiles(n_ref)), each slice >= 512 complex K, S <= 64.
// C4 (n_ref = 4096 -> 384 tiles) keeps S = 1 and with it the bit-identity to the oracle's single
// ascending chain; C2, C3, C5 split (their Y then agrees with the oracle to rounding, ~1e-16).
int zgemm_ksplit(int64_t Mout, int64_t K, int64_t n_ref, int num_sms) {
  if (const char* v = select_env("RID_SKETCH_SPLIT")) {  // tests: force a slice count (1 = unsplit)
    const int s = atoi(v);
    if (s >= 1) return s;
  }
  if (Mout >= 2048 || n_ref <= 0 || K <= 0) return 1;
  const int fr = zgemm_pick_fr(Mout);
  int64_t br = 16 * fr;
#define RID_B_BR(FRV) \
  if (fr == (FRV)) br = 8 * (FRV);
  RID_FR_B(RID_B_BR)
#undef RID_B_BR
  const int64_t tiles = ((n_ref + 63) / 64) * ((2 * Mout + br - 1) / br);
  int64_t s = (2 * (int64_t)num_sms + tiles - 1) / tiles;
  const int64_t smax = K / 512 > 1 ? K / 512 : 1;
  if (s > smax) s = smax;
  if (s > 64) s = 64;
  return s < 1 ? 1 : (int)s;
}

cudaError_t zgemm_ordered(const double2* Rm, int64_t ldr, const double2* Bm, int64_t ldb,
                          double2* C, int64_t ldc, int64_t Mout, int64_t N, int64_t K,
                          int mode, double noise, uint64_t seed, int64_t col0, cudaStream_t st,
                          int ksplit, double2* partial) {
  if (Mout <= 0 || N <= 0) return cudaSuccess;
  ZgemmEpilogue ep{mode, noise, seed, col0, K, 0, 0};
  // QRCP trailing update (mode 2, K = nb <= 16): latency-bound read-modify-write of C, so small
  // register-light CTAs, 2 stages, 3 per SM keep more tiles in flight (measured at C4: update total
  // 2.95 -> 2.36 ms against the sketch tiles; 64-row/4-per-SM 2.55, 32x64/3-per-SM 2.76 ms)
  if (mode == 2) {
    if (zgemm_tma_enabled() && select_env("RID_ZGEMM_TMA_UPDATE"))
      return zgemm_tma_ordered(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, mode, noise, seed, col0, st);
    return launch_cfg<1, 8, 8, 1, 16, 2, 3>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st);
  }
  if (const char* v = experiment_env("RID_ZGEMM_VARIANT")) {  // tile experiments (tools/tune_*.py)
    const int id = atoi(v);
#define RID_V(ID, ...) \
  if (id == ID)        \
    return launch_cfg<__VA_ARGS__>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st, ksplit, partial);
    RID_V(1, 2, 11, 4, 2, 16, 4, 1)   // round-1 first version
    RID_V(2, 1, 11, 8, 1, 16, 3, 3)
    RID_V(3, 1, 17, 8, 1, 16, 4, 2)
    RID_V(4, 1, 3, 8, 1, 16, 3, 4)
    RID_V(5, 4, 8, 4, 2, 16, 4, 1)    // round-1 first generation tile
#undef RID_V
    // in-kernel Philox regeneration of R (REGEN): the key of the R that fill_R generated for this
    // sketch (sketch_key; round 1 passed the product's seed argument, 0 for a sketch, so the
    // regenerated R was another matrix and the results differed — the REGEN runs of
    // profiles/r01_tune_regen_vs_pregen.log)
    if (id >= 10 && id <= 11) {
      ep.seed = sketch_key().seed;
      ep.regen_stream = (int)sketch_key().stream;
      if (id == 10)
        return launch_cfg<2, 11, 4, 2, 16, 3, 2, 1>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st,
                                                     ksplit, partial);
      return launch_cfg<1, 17, 8, 1, 16, 3, 2, 1>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st,
                                                   ksplit, partial);
    }
  }
  if (Mout >= 2048) {  // generation (and any tall product); RID_ZGEMM_TMA=1: the TMA-fed kernel
    if (zgemm_tma_enabled())
      return zgemm_tma_ordered(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, mode, noise, seed, col0, st);
    return launch_cfg<1, 8, 8, 1, 16, 3, 3>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st);
  }
  switch (zgemm_pick_fr(Mout)) {
#define RID_CASE_A(FRV)                                                                        \
  case FRV:                                                                                    \
    return launch_cfg<2, FRV, 4, 2, 16, 3, 2>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st,    \
                                              ksplit, partial);
#define RID_CASE_B(FRV)                                                                        \
  case FRV:                                                                                    \
    return launch_cfg<1, FRV, 8, 1, 16, 3, 2>(Rm, ldr, Bm, ldb, C, ldc, Mout, N, K, ep, st,    \
                                              ksplit, partial);
    RID_FR_A(RID_CASE_A)
    RID_FR_B(RID_CASE_B)
#undef RID_CASE_A
#undef RID_CASE_B
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rid

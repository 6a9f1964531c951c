// rid_internal.h — internal launchers shared by the CUDA translation units of librid.
// Not part of the public C ABI (that is include/rid.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "rid_host.h"

namespace rid {

// Ordered complex GEMM C = Rm · Bm on DMMA (k_zgemm.cu). mode 1 adds noise·E(r, col0 + j) with
// E from Philox stream 3 (generation epilogue); mode 2 computes C = C − Rm · Bm (QRCP trailing
// update).
// ksplit > 1 splits K into slices summed by a fixed-order combine (partial: ksplit*Mout*N elems).
cudaError_t zgemm_ordered(const double2* Rm, int64_t ldr, const double2* Bm, int64_t ldb,
                          double2* C, int64_t ldc, int64_t Mout, int64_t N, int64_t K, int mode,
                          double noise, uint64_t seed, int64_t col0, cudaStream_t st,
                          int ksplit = 1, double2* partial = nullptr);
int zgemm_pick_fr(int64_t Mout);
// The same ordered product with TMA-fed, mbarrier-pipelined stages (k_zgemm_tma.cu; bit-identical
// chains), used by zgemm_ordered for tall products (Mout >= 2048: the generation) when
// RID_ZGEMM_TMA=1 (measured no faster; see k_zgemm_tma.cu).
bool zgemm_tma_enabled();
cudaError_t zgemm_tma_ordered(const double2* Rm, int64_t ldr, const double2* Bm, int64_t ldb,
                              double2* C, int64_t ldc, int64_t Mout, int64_t N, int64_t K,
                              int mode, double noise, uint64_t seed, int64_t col0,
                              cudaStream_t st);
// The sketch as three real products (Gauss), 6·l·m·n flops (k_zgemm3m.cu); split-K as above.
// Rs = Re R + Im R (l x m doubles, leading dimension rsum_ld(l), pad rows zero) from rsum_fill;
// Rs == nullptr selects tiles that form the sums in registers.
cudaError_t zgemm3m(const double2* Rm, int64_t ldr, const double* Rs, int64_t ldrs,
                    const double2* Bm, int64_t ldb, double2* C, int64_t ldc, int64_t Mout,
                    int64_t N, int64_t K, cudaStream_t st, int ksplit, double2* partial);
int zgemm3m_ksplit(int64_t Mout, int64_t K, int64_t n_ref, int num_sms);
// The same product with TMA-fed, mbarrier-pipelined stages (k_zgemm3m_tma.cu); used by zgemm3m
// for the tile sizes it covers (zgemm3m_tma_enabled) unless RID_Z3_TMA=0. Bit-identical results.
int zgemm3m_tile_rows(int64_t Mout);
bool zgemm3m_tma_enabled(int64_t Mout);
cudaError_t zgemm3m_tma_rows(const double2* Rm, int64_t ldr, const double* Rs, int64_t ldrs,
                             const double2* Bm, int64_t ldb, double2* C, int64_t ldc, int64_t Mout,
                             int64_t N, int64_t K, cudaStream_t st, int ksplit, double2* partial,
                             int rows);
cudaError_t zgemm3m_tma(const double2* Rm, int64_t ldr, const double* Rs, int64_t ldrs,
                        const double2* Bm, int64_t ldb, double2* C, int64_t ldc, int64_t Mout,
                        int64_t N, int64_t K, cudaStream_t st, int ksplit, double2* partial);
// Up to kZ3BatchMax independent products C_z (mout[z] x N) = Rm_z · Bm_z (K each) in one launch
// (blockIdx.z = z; element offsets from the base pointers; the SRFT's residue GEMMs).
constexpr int kZ3BatchMax = 16;
struct Z3Batch {
  int n;
  int64_t roff[kZ3BatchMax], boff[kZ3BatchMax], coff[kZ3BatchMax], mout[kZ3BatchMax];
  // row of product z's first row in the Re + Im plane (TMA kernel with a plane only; it must be
  // even: a non-swizzled box of doubles starts on a 16-byte boundary)
  int64_t soff[kZ3BatchMax];
};
cudaError_t zgemm3m_batched(const double2* Rm, int64_t ldr, const double2* Bm, int64_t ldb,
                            double2* C, int64_t ldc, const Z3Batch& bt, int64_t N, int64_t K,
                            cudaStream_t st);
// The same on the TMA kernel (k_zgemm3m_tma.cu): Rm holds Mtot rows, Bm holds Nb columns in all.
cudaError_t zgemm3m_tma_batched(const double2* Rm, int64_t ldr, int64_t Mtot, const double2* Bm,
                                int64_t ldb, int64_t Nb, double2* C, int64_t ldc,
                                const Z3Batch& bt, int64_t N, int64_t K, cudaStream_t st);
cudaError_t zgemm3m_tma_batched_h(const double2* Rm, int64_t ldr, int64_t Mtot, const double2* Bm,
                                  int64_t ldb, int64_t Nb, double2* C, int64_t ldc,
                                  const Z3Batch& bt, int64_t N, int64_t K, int rows,
                                  cudaStream_t st, const double* Rs = nullptr, int64_t ldrs = 0,
                                  int64_t Ms = 0);
inline int64_t rsum_ld(int64_t l) { return (l + 1) / 2 * 2; }
cudaError_t rsum_fill(const double2* R, int64_t l, int64_t m, int64_t ldr, double* Rs,
                      int64_t ldrs, cudaStream_t st);
// Sketch dispatch: 3 (Gauss, default) or 4 (ordered real embedding, RID_SKETCH_4M=1) real
// products per complex multiply-add. Rs is only read by the 3M kernel (may be null for 4M).
int sketch_mults();
int sketch_ksplit(int64_t l, int64_t m, int64_t n_ref, int num_sms);
// Columns [col0, col0 + ncols) of the global m x n matrix: with ksplit == 1 the trailing global
// columns of the last, nearly empty wave (sketch_tail) are computed with a K split (partial must
// hold sketch_partial_elems(...) elements).
struct SketchTail {
  int64_t cols;  // trailing global columns computed with the split
  int S;
};
SketchTail sketch_tail(int64_t l, int64_t m, int64_t n, int num_sms);
int64_t sketch_partial_elems(int64_t l, int64_t m, int64_t n, int64_t ncols, int num_sms);
// aux (nullable): a second stream and two events for running the tail set concurrently
struct SketchAux {
  cudaStream_t stream;
  cudaEvent_t fork, join;
};
cudaError_t sketch_gemm(const double2* R, int64_t ldr, const double* Rs, const double2* A,
                        int64_t lda, double2* Y, int64_t ldy, int64_t l, int64_t ncols, int64_t m,
                        cudaStream_t st, int ksplit, double2* partial, int64_t col0, int64_t n,
                        int num_sms, int* launches, const SketchAux* aux = nullptr);
// The sketch with one level of Strassen over Gauss's 3M (k_strassen.cu, R32): planned
// from (l, m, n) only; then every column block passed must start and end on multiples of 64.
bool strassen_enabled();
bool strassen_plan(int64_t l, int64_t m, int64_t n, int num_sms);
int strassen_ksplit(int64_t l, int64_t m, int64_t n, int num_sms);  // K slices, from (l, m, n)
struct StrassenWs {
  int64_t ldc, lds;                 // leading dimensions of Rc (complex) and Rs (double)
  size_t rc_bytes, rs_bytes, m_bytes;
};
StrassenWs strassen_ws(int64_t l, int64_t m, int64_t ncols);
// Rc / Rs: the seven R combinations (7 l/2 rows x m/2) and their Re + Im planes, from R (l x m)
cudaError_t strassen_rcomb(const double2* R, int64_t l, int64_t m, int64_t ldr, double2* Rc,
                           int64_t ldc, double* Rs, int64_t lds, cudaStream_t st);
// Y (l x ncols, ncols % 64 == 0) = R A for a 64-aligned column block; M: S * m_bytes of workspace
// (S = strassen_ksplit of the whole matrix's (l, m, n))
cudaError_t strassen_sketch(const double2* Rc, int64_t ldc, const double* Rs, int64_t lds,
                            const double2* A, int64_t lda, double2* Y, int64_t ldy, int64_t l,
                            int64_t ncols, int64_t m, double2* M, int S, cudaStream_t st,
                            const SketchAux* aux, int* launches);
// K slices for a sketch of Mout rows, K = m, chosen from n_ref = n_global / 8 only (G-invariant)
int zgemm_ksplit(int64_t Mout, int64_t K, int64_t n_ref, int num_sms);

// The Philox key (seed, stream) of the sketch matrix R most recently generated on this thread
// (rid_api.cu fill_R): read only by the in-kernel regeneration experiment (RID_ZGEMM_VARIANT=10/11).
struct SketchKey {
  uint64_t seed = 0;
  uint32_t stream = 4;
};
inline SketchKey& sketch_key() {
  static thread_local SketchKey k;
  return k;
}

// out(i, j) = N(seed, s, row0 + i, col0 + j), column-major with leading dimension ld (k_misc.cu)
cudaError_t normal_fill(uint64_t seed, uint32_t s, int64_t rows, int64_t cols, int64_t row0,
                        int64_t col0, double2* out, int64_t ld, cudaStream_t st);

// Column-pivoted Householder QR of Y (l x n, in place), k steps (k_qrcp.cu).
struct QrcpOut {
  int64_t* J;        // device, k
  double* beta;      // device, k: R11 diagonal (real)
  double* resid;     // device, k: nu_p at each step
  double* margin;    // device, k: (nu(1) - nu(2)) / nu(1) at each step
  int* info;         // device, 2: [0] status (0 ok, 2 rank failure), [1] rank achieved
  double2* R11;      // device, k x k column-major: the pivot triangle (column s = step s)
};
struct QrcpWork {
  double* nu;        // n: current residual norms (-1 = chosen)
  double* cand;      // 2 * 8 * max_blocks doubles: per CTA (best, second, index-as-double) or the
                     // lazy kernel's 64-byte (b1, b2, b3, m, index) records, x 2 parities
  unsigned* bar;     // 1
  int max_blocks;
  unsigned long long* trace = nullptr;  // optional: 4 %globaltimer stamps per step (CTA 0)
  // blocked variant (k_qrcp_panel)
  double* nuref = nullptr;  // n: norm at the last exact computation (downdating safeguard)
  double* scal = nullptr;   // 1: max_c ||Y[:, c]||
  double2* V = nullptr;     // l x kNB: the panel's reflectors (column-major, ld = l)
  double2* F = nullptr;     // kNB x n: f_s(c) (column-major, ld = kNB)
  double2* Dd = nullptr;    // kNB x n: d_s(c) = v_sᴴ y(c) of the panel (lazy kernel)
  // shared-memory-resident exact kernel (k_qrcp_smem)
  double2* xslot = nullptr; // 2 x max_blocks x l: each CTA's best column, by step parity
};
// one workspace buffer of qrcp_work_bytes(n, l, max_blocks) bytes, carved by qrcp_work_carve
size_t qrcp_work_bytes(int64_t n, int64_t l, int max_blocks);
QrcpWork qrcp_work_carve(void* buf, int64_t n, int64_t l, int max_blocks);
// variant: 1 = blocked panels + tensor-core trailing update (default), 0 = exact recompute
// every step (one persistent kernel). *launches += kernels enqueued.
cudaError_t qrcp(double2* Y, int64_t ldy, int64_t l, int64_t n, int64_t k, double tol_rel,
                 const QrcpOut& out, const QrcpWork& w, int num_sms, cudaStream_t st,
                 int* launches, int variant = -1);

// The sharded QR: the sketch of an n-column matrix held as G column
// blocks, rank g's block (global columns [g n_loc, (g + 1) n_loc)) in its own buffer Y[g] with its
// own workspace w[g] (nu, nuref, F sized n_loc; V; scal), factored by the blocked kernel with the
// CTAs split into G rank groups: rank g's CTAs touch only rank g's columns, and across ranks only
// the per-CTA pivot candidates (w[0].cand, one grid barrier per step) and, per step, the pivot
// column (rows j..l-1 plus its k_NB pending-reflector coefficients, read from the owner's block)
// move. Every rank's outputs out[g] (J in GLOBAL ids, beta, resid, margin, info, R11) are written
// and identical. G = 1 is qrcp()'s blocked path: the same kernel, bitwise the same results for any
// G (every column's arithmetic and the pivot reduction are independent of the sharding).
constexpr int kQrMaxRanks = 8;
struct QrShards {
  int G = 1;
  int64_t n_loc = 0;
  double2* Y[kQrMaxRanks] = {};
  QrcpOut out[kQrMaxRanks] = {};
  QrcpWork w[kQrMaxRanks] = {};
};
// one cooperative launch per panel over all G blocks (the one-GPU form; the real multi-GPU
// transport is not built: DESIGN.md §8.2), plus G tensor-core trailing updates per panel
cudaError_t qrcp_sharded(const QrShards& sh, int64_t ldy, int64_t l, int64_t k, double tol_rel,
                         int num_sms, cudaStream_t st, int* launches);

// The paper's QR: column-pivoted CGS with one reorthogonalisation (k_cgs2.cu).
// Same outputs as qrcp (J, beta, resid, margin, info, R11) and the same contract on Y: on return
// Y[0:k, c] = R[:, c] with R = Q^H Y (the rows below k are left as they were).
size_t cgs2_work_bytes(int64_t l, int64_t n, int64_t k, int num_sms);
cudaError_t cgs2(double2* Y, int64_t ldy, int64_t l, int64_t n, int64_t k, double tol_rel,
                 const QrcpOut& out, void* work, int num_sms, cudaStream_t st, int* launches,
                 unsigned long long* trace = nullptr);

// Inverse of the pivoted triangle R11 (R11[t, s] = Y[t, J[s]] for t < s, beta[s] on the diagonal)
cudaError_t tri_inverse(const double2* R11, int64_t k, double2* Rinv, cudaStream_t st);
// P[:, J_t - col0] = e_t for pivots inside the shard (k_misc.cu)
cudaError_t assemble_identity(const int64_t* J, int64_t k, int64_t col0, int64_t n_loc, double2* P,
                              int64_t ldp, cudaStream_t st);
// B(:, t) = A(:, J_t - col0) for pivots inside the shard (k_misc.cu); a J_t outside [0, n) sets
// *bad (device int) and leaves column t untouched
cudaError_t gather_columns(const double2* A, int64_t lda, int64_t m, const int64_t* J, int64_t k,
                           int64_t col0, int64_t n_loc, int64_t n, double2* B, int64_t ldb,
                           int* bad, cudaStream_t st);
// dst = sum over g < G of src.p[g], elementwise, added in rank order (k_misc.cu)
constexpr int kMaxLocalRanks = 64;
struct RankPtrs {
  const double* p[kMaxLocalRanks];
};
cudaError_t sum_ranks(const RankPtrs& src, int G, double* dst, int64_t count, cudaStream_t st);

// Compensated power-iteration pieces (k_estimate.cu). Vectors of "cdd" are 4 doubles per entry
// (re.s, re.c, im.s, im.c): a Dot2 accumulator whose value is s + c.
struct EstPlan {
  bool tma;  // TMA-fed passes (k_ax_tma / k_z_tma; RID_EST_TMA=0 selects k_ax / k_z)
  int64_t px_chunk;
  int px_parts;
  int64_t ax_split_cols;
  int ax_parts;
  int ax_rblocks;  // row blocks of 128 (TMA pass)
  int z_blocks;
  int x0_blocks;
  int num_sms;
};
EstPlan est_plan(int64_t m, int64_t n_loc, int64_t k, int num_sms);
cudaError_t est_x0(uint64_t seed, int64_t col0, int64_t n_loc, double2* x, double* part,
                   const EstPlan& p, cudaStream_t st);
cudaError_t est_merge_scalar(const double* part, int nparts, double* out, cudaStream_t st);
// vmax: max |re| + |im| of the produced vector (atomicMax on the bits; zeroed by the launcher),
// with amax (from the first A x pass) the bounds of the fixed-offset accumulation
cudaError_t est_normalise(const double2* v, int64_t n_loc, const double* nn, double2* x,
                          double* est_out, unsigned long long* vmax, cudaStream_t st);
cudaError_t est_px(const double2* P, int64_t ldp, int64_t k, int64_t n_loc, const double2* x,
                   double* part, double* u_out, const EstPlan& p, cudaStream_t st);
cudaError_t est_merge_vec(const double* part, int nparts, int64_t len, double* out,
                          cudaStream_t st);
// bounds = {amax, xmax} (est_ax) / {amax, ymax} (est_z), device
// first = true: the first iteration's pass, Dot2 and recording amax into bounds[0]
cudaError_t est_ax(const double2* A, int64_t lda, int64_t m, int64_t n_loc, const double2* x,
                   unsigned long long* bounds, double* part, const EstPlan& p, cudaStream_t st,
                   bool first = false);
cudaError_t est_y(const double* wpart, int nparts, int64_t m, const double2* B, int64_t ldb,
                  int64_t k, const double* u, double2* y, unsigned long long* vmax,
                  cudaStream_t st);
cudaError_t est_bhy(const double2* B, int64_t ldb, int64_t m, int64_t k, const double2* y,
                    double* sb, cudaStream_t st);
cudaError_t est_z(const double2* A, int64_t lda, int64_t m, int64_t n_loc, const double2* y,
                  const double2* P, int64_t ldp, int64_t k, const double* sb, double2* z,
                  const unsigned long long* bounds, double* npart, const EstPlan& p,
                  cudaStream_t st);

}  // namespace rid

namespace rid {
// SRFT randomisation Y = S F D A (k_srft.cu). m a power of two, m >= 16.
size_t srft_work_bytes(int64_t m, int64_t l, int64_t n_loc);
cudaError_t srft_sketch(uint64_t seed, bool retry, int64_t l, const double2* A, int64_t m,
                        int64_t n, int64_t n_loc, int64_t lda, double2* Y, int64_t ldy, void* work,
                        double2* splitk, size_t splitk_elems, int num_sms, cudaStream_t st,
                        int* launches);
}  // namespace rid

namespace rid {
// The sketch as an exact modular integer product on the int8 tensor cores (k_crt.cu, DESIGN.md
// §5.5): T moduli, b-bit operands, K' = 2 mh split into kslices of kbps 128-byte blocks (int32
// exact), the l rows in `chunks` tiles of nc (TMEM columns), lp = chunks * nc.
struct CrtPlan {
  int T, b, kslices, kbps, chunks, nc;
  int64_t mh, Kp, lp;
  bool pair;  // the CTA-pair GEMM (k_imma2, tcgen05 cta_group::2; N a multiple of 32)
  int cn[8], coff[8];  // row tile c: cn[c] rows from row coff[c] (nc = the largest)
};
CrtPlan crt_plan(int64_t l, int64_t m);
void crt_balance(CrtPlan& p, int64_t ncols, int num_sms);  // extra K slices for wave balance
int crt_moduli(int* p, int cap);
double crt_log2M(int T);
size_t crt_R_bytes(const CrtPlan& p);                  // R's residue operands + row maxima
size_t crt_A_bytes(const CrtPlan& p, int64_t ncols);  // one column block's residues + outputs
cudaError_t crt_prep_R(const CrtPlan& p, const double2* R, int64_t ldr, int64_t l, int64_t m,
                       void* wsR, cudaStream_t st, int* launches);
// the column-block pipeline's second stream and events (created by the caller)
struct CrtPipe {
  cudaStream_t stream;
  cudaEvent_t fork, join, prep[2], gemm[2];
};
// events recorded around each GEMM launch (ev[2 g], ev[2 g + 1] for launch g < nev / 2; external
// records while a graph is captured); `used` = GEMM launches timed by the last call
struct CrtTiming {
  cudaEvent_t* ev;
  int nev;
  bool external;
  mutable int used;
};
// columns per block for a workspace budget (bytes per block buffer)
int64_t crt_block_cols(const CrtPlan& p, int64_t ncols, int64_t budget_bytes, int num_sms);
// Y (l x ncols) = R A: column blocks of <= nb columns, ws[0], ws[1] of crt_A_bytes(p, nb) each
// (ws[1] unused when pipe == nullptr: one stream, one buffer)
cudaError_t crt_sketch(const CrtPlan& p, const void* wsR, const double2* A, int64_t lda, double2* Y,
                       int64_t ldy, int64_t l, int64_t ncols, int64_t m, void* const ws[2],
                       int64_t nb, int num_sms, cudaStream_t st, const CrtPipe* pipe,
                       const CrtTiming* tim, int* launches);
}  // namespace rid

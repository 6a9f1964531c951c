/*
 * rid.h — C ABI of librid: the randomized interpolative decomposition (ID) of
 * Lucas, Stalzer & Feo, "Parallel implementation of fast randomized algorithms for the
 * decomposition of low rank matrices" (arXiv 1205.3830), on NVIDIA B200 (sm_100a).
 *
 * Problem (§2, Eq. 1): given a complex m x n matrix A of approximate rank k, find
 * k column indices J (B = A[:, J]) and a k x n matrix P with A ≈ B P. The randomised algorithm
 * (§2) sketches Y = R A with an l x m random R (l = k + oversampling), factors
 * Y ≈ Q [R1 R2] with a column permutation, solves R2 = R1 T and sets P = [I T].
 *
 * Conventions for every call
 *   - complex values are IEEE binary64 pairs (re, im) ("rid_z", 16 bytes, = cuDoubleComplex =
 *     torch.complex128 element); matrices are COLUMN-MAJOR with a leading dimension ld ≥ rows.
 *   - A column shard is columns [col0, col0 + n_loc) of the global m x n matrix A. With a
 *     communicator of G ranks, rank g holds one contiguous shard and every rank calls
 *     collectively with the same (m, n, k, l, seed, ...).
 *   - Pointers may be DEVICE pointers (on the context's device) or HOST pointers (pageable or
 *     pinned). The library detects which (cudaPointerGetAttributes); host buffers are staged
 *     through device workspace with the copies on the context stream (this is the "e2e" path).
 *   - Ownership: the caller owns every buffer passed in; the library never retains a caller
 *     pointer after a call returns. The library owns transient workspace inside the context
 *     (sketch matrix R, the full Y, reflectors, B = A[:, J], estimator vectors) and frees it in
 *     rid_destroy.
 *   - Calls are ordered on the context stream. rid_generate and rid_sketch return after
 *     enqueueing when all buffers are on the device; rid_decompose and rid_error_estimate
 *     synchronise the stream once (to read the rank status / the estimate). Any call with host
 *     buffers synchronises before returning.
 *   - Errors: a status code is returned; no exception or abort crosses the ABI; the message is in
 *     rid_last_error(ctx). Argument errors (RID_EINVAL) are detected before anything is enqueued.
 *
 * Randomness: every random matrix entry is N(seed, s, i, j) of docs/RNG.md (Philox4x32-10 with
 * counter (i, j, s, 0), key = seed; complex Gaussian with parts N(0, 1/2)): X s=1, Y0 s=2,
 * E s=3, R s=4 (s=20 on the one retry), estimator start vector s=5.
 */
#ifndef RID_H_
#define RID_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double re, im;
} rid_z;

typedef enum {
  RID_OK = 0,
  RID_EINVAL = 1,     /* argument violates a precondition (nothing was enqueued) */
  RID_ERANK = 2,      /* sketch rank < k after one re-randomisation */
  RID_ESINGULAR = 3,  /* |R11[i,i]| < 1e-13 max |R11 diag| */
  RID_ENOMEM = 4,     /* device or pinned allocation failed */
  RID_ECUDA = 5,      /* a CUDA runtime error; see rid_last_error */
  RID_ENCCL = 6       /* an NCCL error; see rid_last_error */
} rid_status;

typedef struct rid_ctx rid_ctx;

/* Randomisation used by rid_decompose (rid_set_sketch). */
typedef enum {
  RID_SKETCH_GAUSSIAN = 0, /* Y = R A, R l x m complex Gaussian (north star; default)            */
  RID_SKETCH_SRFT = 1      /* Y = S F D A (Eqs. 4–7); m a power of two >= 16     */
} rid_sketch_kind;

/* Arithmetic of the Gaussian sketch Y = R A (rid_set_sketch_engine). Both meet the north-star bar
 * (Y within 1e-12 relative Frobenius of the oracle; measured ~4e-14); J and P follow from Y. */
typedef enum {
  RID_ENGINE_AUTO = 0,     /* INT8_CRT when l m n >= 2^34 (C3-C5), else FP64_DMMA (default); the
                              INT8_CRT engine takes l <= 2048 and m <= 2^28 (else FP64_DMMA)       */
  RID_ENGINE_FP64_DMMA = 1,/* complex128 products on the FP64 tensor pipe (DMMA.8x8x4: Gauss 3M,
                              one Strassen level over it for the unsplit plans)                    */
  RID_ENGINE_INT8_CRT = 2  /* the exact integer product of R and A rounded to b bits relative to
                              their row / column maxima, computed as T int8 GEMMs on tcgen05 (one
                              per modulus) and recovered by the Chinese remainder theorem
                              (reading R33)                                       */
} rid_sketch_engine;

/* Pivoted QR of the sketch used by rid_decompose, rid_qrcp and rid_factor_solve (rid_set_qr).
 * Both choose the same columns (the greedy largest-residual pivot of PAPER.md:82-86) and agree on
 * R = Q^H Y to rounding. */
typedef enum {
  RID_QR_HOUSEHOLDER = 0, /* Householder QRCP (default; the cheaper choice PAPER.md:108 names)    */
  RID_QR_CGS2 = 1         /* classical Gram-Schmidt with one reorthogonalisation, the paper's own
                             QR ("CGS with iteration"); exact norms every step     */
} rid_qr_kind;

/* How rid_decompose factors the sketch when a communicator of G > 1 ranks is set
 * (rid_set_qr_dist). Both give the same J and P bits as one rank. */
typedef enum {
  RID_QR_REPLICATED = 0, /* all-gather Y (16 l n bytes), then every rank factors the whole l x n
                            sketch (default)                                     */
  RID_QR_SHARDED = 1     /* no all-gather: rank g keeps its l x n/G block and the ranks factor the
                            sketch together, exchanging per pivot step only the pivot candidates
                            and the pivot column. Householder QR, G <= 8;
                            built on the in-process data plane of rid_comm_init_local (one GPU);
                            an NCCL communicator refuses it (RID_EINVAL from rid_decompose).     */
} rid_qr_dist;

/* Per-call diagnostics (SPEC.md:298-302 IdDiagnostics); every field is written by the call that
 * receives it; times are device times from CUDA events on the context stream, in seconds. */
typedef struct {
  double t_rgen;      /* Philox fill of the sketch matrix R                       */
  double t_sketch;    /* Y_loc = R A_loc (DMMA)                                    */
  double t_gather;    /* all-gather of Y over the communicator (0 when G = 1)      */
  double t_qrcp;      /* pivoted Householder QR of Y                               */
  double t_solve;     /* R11^{-1}, T = R11^{-1} R12 (DMMA), P = [I T] assembly      */
  double t_total;     /* whole call, device time                                   */
  double t_h2d, t_d2h;/* host staging copies (e2e path), 0 for device buffers      */
  int retries;        /* 0 or 1 sketch re-randomisations             */
  int rank_achieved;  /* k on success; the achieved rank on RID_ERANK              */
  double tie_margin_min; /* min_j (nu(1) - nu(2)) / nu(1) over the k pivot steps (reading R18) */
  double resid_last;  /* nu_p at the last pivot step (|R11[k-1,k-1]|)              */
  int launches;       /* number of librid CUDA kernels this call launched           */
  double t_sketch_tc; /* INT8_CRT engine: the tcgen05 GEMM launches inside t_sketch (0 otherwise) */
  int sketch_engine;  /* the engine the sketch ran on (RID_ENGINE_FP64_DMMA / _INT8_CRT; 0 SRFT) */
} rid_diag;

/* --- context ------------------------------------------------------------------------------- */
/* Create a context on CUDA device `device` whose calls are ordered on `cuda_stream` (a
 * cudaStream_t owned by the caller; NULL = the legacy default stream, as everywhere in CUDA). */
rid_status rid_create(rid_ctx** ctx, int device, void* cuda_stream);
void rid_destroy(rid_ctx* ctx);
/* Re-bind the context to `cuda_stream` (same meaning as in rid_create): subsequent calls are
 * ordered on it. Work already enqueued stays ordered on the previous stream; the caller orders the
 * two streams if the next call depends on it (the Python binding passes torch's current stream on
 * every call of a default context, so both orders are torch's). */
rid_status rid_set_stream(rid_ctx* ctx, void* cuda_stream);
/* Last error message of this context ("" when none). Valid until the next call on ctx. */
const char* rid_last_error(const rid_ctx* ctx);
/* Library version string and the compiled GPU architecture ("sm_100a"). */
const char* rid_version(void);

/* --- communicator (column sharding over G GPUs, NCCL over NVLink) --------------------------- */
/* Size of the opaque unique-id blob (NCCL_UNIQUE_ID_BYTES). */
size_t rid_comm_id_bytes(void);
/* Rank 0 creates the id (writes rid_comm_id_bytes() bytes to `id`); the caller broadcasts it
 * to the other ranks by any means (the Python layer uses torch.distributed). */
rid_status rid_comm_get_id(void* id);
/* Every rank: join the communicator of `nranks` ranks as `rank` (collective, blocking). */
rid_status rid_comm_init(rid_ctx* ctx, const void* id, int rank, int nranks);
/* In-process communicator over the `nranks` contexts ctxs[0..nranks-1] (one process, ONE device;
 * context r becomes rank r). The collectives of rid_decompose / rid_error_estimate then run as
 * device copies between the contexts' workspaces ordered by CUDA events, with a host rendezvous
 * of the calling threads at each collective: every rank's calls must be made concurrently from
 * its own host thread (exactly as with NCCL, one thread per rank). This is how the G > 1 data
 * path runs on a machine with fewer GPUs than ranks (tests/test_gpu_multirank.py); results are
 * the same bits as with NCCL (the all-gathers are copies; the one all-reduce, of B = A[:, J],
 * adds one nonzero per element). RID_EINVAL: nranks outside [1, 64], repeated contexts, or
 * contexts on different devices. A rank that does not reach a collective within 300 s makes
 * every rank's call fail with RID_ENCCL. */
rid_status rid_comm_init_local(rid_ctx** ctxs, int nranks);
/* Query: rank and nranks (1, 0 when no communicator). */
rid_status rid_comm_info(const rid_ctx* ctx, int* rank, int* nranks);

/* --- the method ---------------------------------------------------------------------------- */
/* A[:, shard] = X Y0 + noise E (docs/RNG.md §5): X m x k, Y0 k x n, E m x n from
 * Philox. Bit-identical to the CPU oracle. Preconditions: 1 <= k <= min(m, n), 0 <= col0,
 * n_loc >= 0, col0 + n_loc <= n, lda >= m, m, n < 2^32. */
rid_status rid_generate(rid_ctx* ctx, uint64_t seed, int64_t m, int64_t n, int64_t k, double noise,
                        int64_t col0, int64_t n_loc, rid_z* A, int64_t lda);

/* Y (l x n_loc) = R A with R(r, i) = N(seed, stream, r, i) (north_star; PAPER.md:97 licenses the
 * Gaussian sketch in place of the SRFT of Eqs. 4–7). stream is 4 (or 20 on the retry).
 * A is a block of n_loc columns of an m x n matrix (n = n_loc for a whole matrix): n fixes the
 * K-split of the DMMA product (rid_sketch_splits), so the columns of Y are bit-identical for
 * every sharding of the same n. The complex products use Gauss's three real multiplications
 * (rid_sketch_mults() == 3, default; R31): Y agrees with the oracle's ascending chain
 * to rounding (north-star bar 1e-12 relative). With RID_SKETCH_4M=1 in the environment the
 * real embedding with four (rid_sketch_mults() == 4) is used: with one slice its K summation is
 * the ascending fused chain and Y is bit-identical to the oracle's naive loop; with S slices the
 * slice sums are added in slice order. Preconditions: 1 <= l <= m, n_loc <= n, lda >= m,
 * ldy >= l. */
rid_status rid_sketch(rid_ctx* ctx, uint64_t seed, uint32_t stream, int64_t l, const rid_z* A,
                      int64_t m, int64_t n, int64_t n_loc, int64_t lda, rid_z* Y, int64_t ldy);
/* The same for the columns [col0, col0 + n_loc) of the m x n matrix (rid_sketch: col0 = 0).
 * The global position matters to the kernel plan only: when the unsplit sketch's last wave of
 * CTAs would be nearly empty, the trailing global columns that fall into it are computed with a
 * K split (fixed-order slice sums), so every column's bits depend on (m, l, n, its index) alone —
 * identical for every sharding. Preconditions as rid_sketch, plus 0 <= col0, col0 + n_loc <= n. */
rid_status rid_sketch_cols(rid_ctx* ctx, uint64_t seed, uint32_t stream, int64_t l,
                           const rid_z* A, int64_t m, int64_t n, int64_t col0, int64_t n_loc,
                           int64_t lda, rid_z* Y, int64_t ldy);
/* The paper's own randomisation Y = S F D A (§2, Eqs. 4–7; docs/RNG.md §7):
 * D random unit phases (Philox stream 6), F the unnormalised DFT (Eq. 6), S l row samples with
 * replacement (stream 7); retry != 0 uses streams 22/23. Computed as a 16-point DFT
 * pass plus 16 small DMMA GEMMs (8 l m n / 16 flops); agrees with the direct sum to rounding.
 * Preconditions: m a power of two, 16 <= m < 2^32, 1 <= l, n_loc <= n, lda >= m, ldy >= l. */
rid_status rid_sketch_srft(rid_ctx* ctx, uint64_t seed, int retry, int64_t l, const rid_z* A,
                           int64_t m, int64_t n, int64_t n_loc, int64_t lda, rid_z* Y,
                           int64_t ldy);
/* Select the randomisation of subsequent rid_decompose calls on ctx (default GAUSSIAN). */
rid_status rid_set_sketch(rid_ctx* ctx, int kind);
/* Select the arithmetic of subsequent Gaussian sketches on ctx (rid_sketch_engine; default AUTO).
 * RID_SKETCH_CRT=0/1 in the environment overrides it (FP64_DMMA / INT8_CRT). */
rid_status rid_set_sketch_engine(rid_ctx* ctx, int engine);
/* The engine (RID_ENGINE_FP64_DMMA or RID_ENGINE_INT8_CRT) a Gaussian sketch of an m x n matrix
 * with l rows runs on ctx: a function of (m, l, n), the context's selection and the environment. */
int rid_sketch_engine_of(const rid_ctx* ctx, int64_t m, int64_t l, int64_t n);
/* The INT8_CRT plan of an l x m sketch matrix (pure host arithmetic; any pointer may be NULL):
 * T moduli, b bits per operand, kslices K' slices (each exact in int32), Kp = padded K' = 2 m,
 * nc rows of R per tensor-memory tile, log2(prod p_t) in log2M. RID_EINVAL for l < 1, m < 1 or
 * l > 2048 (the engine's limit: larger sketches run on FP64_DMMA whatever the selection). */
rid_status rid_crt_plan(int64_t l, int64_t m, int* T, int* b, int* kslices, int64_t* Kp, int* nc,
                        double* log2M);
/* The moduli of the INT8_CRT engine (up to 16 values written to p; returns how many exist). */
int rid_crt_moduli(int* p, int cap);

/* Select the pivoted QR of subsequent rid_decompose / rid_qrcp / rid_factor_solve calls on ctx
 * (default HOUSEHOLDER). RID_EINVAL for an unknown kind. CGS2 needs a workspace of
 * 16 (2 l n + 2 l k + k n) + 8 l (k + 1) bytes beyond Householder's. */
rid_status rid_set_qr(rid_ctx* ctx, int kind);
/* Select how subsequent rid_decompose calls on ctx factor a sharded sketch (rid_qr_dist; default
 * RID_QR_REPLICATED). Every rank of a communicator must select the same mode. RID_EINVAL for an
 * unknown mode. */
rid_status rid_set_qr_dist(rid_ctx* ctx, int mode);
/* Number of K slices S the sketch of an m-row, n-column matrix uses (1 = unsplit): chosen so that
 * the n/8-column shard of an 8-GPU run still fills the GPU, a function of (m, l, n) only. */
int rid_sketch_splits(const rid_ctx* ctx, int64_t m, int64_t l, int64_t n);
/* 1 when the Gaussian sketch of an m x n matrix with l rows runs one level of Strassen's
 * algorithm over Gauss's three products (R32: 7/8 of the tensor work, 5.25 l m n flop;
 * Y agrees with the oracle to ~1e-14 relative), 0 otherwise. A function of (m, l, n) only:
 * l % 4 == 0, l >= 64, m % 32 == 0, m >= 1024, n % 512 == 0 (C2-C5), and RID_SKETCH_STRASSEN != 0
 * in the environment. When it is 1, every column block passed to rid_sketch_cols / rid_decompose
 * must start and end on a multiple of 64 (RID_EINVAL otherwise; every G <= 8 dividing n gives such
 * shards): the algorithm pairs the two 32-column halves of each aligned 64-column group. */
int rid_sketch_strassen(const rid_ctx* ctx, int64_t m, int64_t l, int64_t n);
/* Real multiplications per complex multiply-add in the sketch kernel: 3 (Gauss, 6 l m n flops,
 * default) or 4 (real embedding, 8 l m n flops, bit-exact ordered chain; RID_SKETCH_4M=1). */
int rid_sketch_mults(void);

/* The whole ID on a column shard: sketch -> all-gather Y -> column-pivoted
 * Householder QR of Y (k steps, greedy max-norm pivot, ties -> lowest index) -> T = R11^{-1} R12
 * for the local columns -> P_loc = [I T] in original column order (P[t, J_t] = 1 exactly).
 * Outputs: J (k int64, GLOBAL column ids in pivot order; replicated on every rank) and P_loc
 * (k x n_loc, ldp >= k). On RID_ERANK after one retry with R stream 20, J/P are unspecified.
 * Preconditions: 1 <= k <= min(m, n), k <= l <= min(m, 2048), shard as for rid_generate,
 * G * n_loc == n when a communicator is set. diag may be NULL. */
rid_status rid_decompose(rid_ctx* ctx, const rid_z* A, int64_t m, int64_t n, int64_t col0,
                         int64_t n_loc, int64_t lda, int64_t k, int64_t l, uint64_t seed,
                         int64_t* J, rid_z* P, int64_t ldp, rid_diag* diag);

/* Power-iteration estimate of ||A - A[:, J] P||_2 (Table 5): x0 from stream 5
 * normalised, q fixed iterations of y = A x - B (P x), z = A^H y - P^H (B^H y), est = sqrt(||z||),
 * x = z / ||z||, with compensated accumulation in every dot product: TwoProd + TwoSum (Dot2), and
 * in the two streaming passes over A TwoProd + Fast2Sum against a power-of-two offset above a
 * bound from max|A| (recorded by the first iteration's pass, which runs Dot2) and max|x| / max|y|
 * (error-free as well; R16').
 * J are global column ids (as returned by rid_decompose), P the local k x n_loc block.
 * *est is written on the host. Preconditions: q >= 1, shapes as above. */
rid_status rid_error_estimate(rid_ctx* ctx, const rid_z* A, int64_t m, int64_t n, int64_t col0,
                              int64_t n_loc, int64_t lda, const int64_t* J, int64_t k,
                              const rid_z* P, int64_t ldp, int q, uint64_t seed, double* est,
                              rid_diag* diag);

/* Eq. (3) right-hand side 50 sqrt(mn) (1/eps)^(1/k) sigma_kp1. Host only. */
double rid_error_bound(int64_t m, int64_t n, int64_t k, double eps, double sigma_kp1);

/* --- lower-level entry points (the steps of rid_decompose, for tests and G-emulation) --------- */
/* out(i, j) = N(seed, s, row0 + i, col0 + j), rows x cols, leading dimension ld. */
rid_status rid_normal_fill(rid_ctx* ctx, uint64_t seed, uint32_t s, int64_t rows, int64_t cols,
                           int64_t row0, int64_t col0, rid_z* out, int64_t ld);
/* Pivoted QR of a full sketch Y (l x n, copied; the caller's Y is not modified). Outputs J (k),
 * R (k x n, original column order: R[:, c] = Q^H Y[:, c] rows 0..k-1, zero below the diagonal of
 * the pivot columns), resid (k, nu_p per step) and margin (k, tie margins); any of R, resid,
 * margin may be NULL. Returns RID_ERANK with diag->rank_achieved on rank failure. */
rid_status rid_qrcp(rid_ctx* ctx, const rid_z* Y, int64_t l, int64_t n, int64_t ldy, int64_t k,
                    int64_t* J, rid_z* R, int64_t ldr, double* resid, double* margin,
                    rid_diag* diag);
/* P_loc from a full sketch Y (l x n): the factorisation of rid_qrcp followed by the solve for
 * columns [col0, col0 + n_loc). Used to emulate G shards on one GPU. */
rid_status rid_factor_solve(rid_ctx* ctx, const rid_z* Y, int64_t l, int64_t n, int64_t ldy,
                            int64_t k, int64_t col0, int64_t n_loc, int64_t* J, rid_z* P,
                            int64_t ldp, rid_diag* diag);

#ifdef __cplusplus
}
#endif
#endif /* RID_H_ */

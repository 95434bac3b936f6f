/*
 * kpm.h -- C ABI of the B200-native KPM-DOS hot path (arXiv:1410.5242).
 *
 * The library computes the Chebyshev moments of the Kernel Polynomial Method with the
 * blocked, augmented SpMMV of Fig. 5 `alg:kpm_improved_blocked`:
 * every sweep applies H~ = a(H - b 1) to a row-major block of R vectors, forms
 * W <- 2 H~ V - W and the two column-wise scalar products eta_2m = <V|V>,
 * eta_2m+1 = <W|V> in the same pass over the matrix, so the
 * matrix is read M/2 times in total.  Moments are reduced across ranks once, at
 * the end (Table III).
 *
 * Conventions shared by every entry point
 *   - Every function returns kpm_status; nothing throws across the ABI.
 *   - Complex numbers are interleaved (re, im) doubles.  Block vectors are row-major:
 *     element (i, r) of an n x R block is at index i*R + r.
 *   - The caller owns every pointer it passes and may free it when the call returns
 *     (kpm_set_matrix copies the matrix).  The library owns all device memory it
 *     allocates; kpm_destroy releases it.
 *   - Host pointers are plain pageable or pinned memory.  KPM_MEM_DEVICE inputs are
 *     device pointers on the context's device.
 *   - On an error the context stays usable, except after KPM_ECUDA / KPM_ENCCL, after
 *     which only kpm_destroy and kpm_last_error are valid.
 *   - One host thread per context at a time.
 *   - nranks > 1 (NCCL): kpm_moments* and the setup collectives poll NCCL's asynchronous error
 *     state while they wait for the device; an error NCCL reports aborts the communicator and
 *     returns KPM_ENCCL.  A peer that dies silently is not detected (no watchdog).
 *   - nranks > 1: kpm_create, kpm_set_matrix and kpm_moments* are collective: every rank
 *     calls them in the same order with identical n_global, a, b, M, R, seed; the row
 *     ranges [row_begin, row_end) tile [0, n_global) in rank order (the data-parallel
 *     row distribution of P:849-854, equal weights).
 */
#ifndef KPM_H
#define KPM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kpm_ctx kpm_ctx; /* opaque, owned by the library */

typedef enum {
  KPM_OK = 0,
  KPM_EINVAL = 1,     /* bad argument: M odd or < 2, R < 1, a <= 0, non-finite a/b/values,
                         NULL pointer, malformed CSR, unsupported option                 */
  KPM_ESTATE = 2,     /* kpm_moments* before kpm_set_matrix                                 */
  KPM_ERANGE = 3,     /* local rows + halo rows > INT32_MAX (4-byte kernel indices),
                         or a column outside [0, n_global)                                 */
  KPM_ENOMEM = 4,     /* device or host allocation failed                                   */
  KPM_ECUDA = 5,      /* CUDA error (sticky: destroy the context)                           */
  KPM_ENCCL = 6,      /* NCCL error (sticky)                                                */
  KPM_EZERONORM = 7,  /* kpm_moments_v0: a start column has eta_0 = <v|v> = 0               */
  KPM_WDIVERGED = 8   /* warning, results written: some |mu_n| > mu_0 (1 + 1e-8), i.e. a, b do
                         not map the spectrum into [-1, 1]                          */
} kpm_status;

enum { KPM_MEM_HOST = 0, KPM_MEM_DEVICE = 1 };

typedef struct {
  int device;                   /* CUDA device ordinal of this rank                         */
  int nranks;                   /* >= 1                                                     */
  int rank;                     /* 0 .. nranks-1                                            */
  const void* nccl_unique_id;   /* 128-byte ncclUniqueId, identical on all ranks; NULL when
                                   nranks == 1                                              */
  void* cuda_stream;            /* cudaStream_t every kernel and copy is issued on, or NULL
                                   for a library-owned stream                               */
  int sell_C;                   /* SELL chunk height C; 0 -> 32. Only 32 (= warpSize)
                                   is supported                                             */
  int sell_sigma;               /* SELL sorting scope sigma; 0 -> 1 (no sorting). 1 or a
                                   multiple of C                                            */
  unsigned flags;               /* 0 or an OR of the KPM_* option flags below               */
} kpm_options;

/* kpm_options.flags: KPM_CHECK_HERMITIAN makes kpm_set_matrix verify H_ij == conj(H_ji)
 * (|difference| <= 1e-12 max|H_kl|, duplicates summed, a missing partner counting as 0) over
 * the entries whose row and column both belong to this rank -- a debug aid, O(nnz log nnz) on
 * the host; KPM_EINVAL naming the first offending pair otherwise.  The method needs a
 * Hermitian H (the eta -> mu doubling identities). */
enum { KPM_CHECK_HERMITIAN = 1u };
/* KPM_DETERMINISTIC: accepted for SURVEY §8(b) compatibility; the library is always
 *   deterministic (fixed chunk -> CTA map, fixed-order CTA and grid sums, no floating-point
 *   atomics: bitwise identical moments run to run for a fixed nranks, R and kernel variant).
 * KPM_TIMING: kpm_moments* record a CUDA event after every sweep (and launch the sweeps one by
 *   one instead of replaying a CUDA graph); kpm_last_sweep_times returns the per-sweep times.
 * KPM_VIRTUAL_RANKS: test harness.  nranks contexts on ONE device, one host thread each, form an
 *   in-process group: nccl_unique_id must point to a kpm_vgroup (kpm_vgroup_create) instead of
 *   an NCCL id.  Setup collectives and the final eta reduction run on the host through the
 *   group; the halo exchange is the fused one (peer stores from the edge kernels' epilogue,
 *   flag epochs) with plain device pointers in place of CUDA IPC mappings.  Every sweep kernel
 *   and the edge / interior split are the multi-GPU ones, so a single-GPU box can test them.
 *   Needs CUDA_DEVICE_MAX_CONNECTIONS >= 2 * nranks set before CUDA starts (every rank's stream
 *   can block on another rank's flag; streams must not share a hardware queue), else
 *   kpm_create returns KPM_EINVAL. */
enum { KPM_DETERMINISTIC = 2u, KPM_TIMING = 4u, KPM_VIRTUAL_RANKS = 8u };

typedef struct kpm_vgroup kpm_vgroup; /* opaque in-process rank group (KPM_VIRTUAL_RANKS) */
/* Create / destroy a group of nranks virtual ranks.  The group must outlive its contexts. */
kpm_status kpm_vgroup_create(int nranks, kpm_vgroup** out);
void kpm_vgroup_destroy(kpm_vgroup* group);

typedef struct {
  int64_t n_global;             /* matrix dimension N                               */
  int64_t row_begin, row_end;   /* this rank's rows [row_begin, row_end)                    */
  const int64_t* row_ptr;       /* row_end-row_begin+1 entries, row_ptr[0] == 0, non-decreasing */
  const int64_t* col;           /* row_ptr[last] global column ids, in [0, n_global); any
                                   order inside a row (the summation order: the row's
                                   diagonal entry, if stored, first, then this order)       */
  const double* val;            /* 2*row_ptr[last] doubles, interleaved (re, im)            */
  int mem;                      /* KPM_MEM_HOST or KPM_MEM_DEVICE (all three arrays)        */
} kpm_csr;

/* A fresh 128-byte NCCL unique id for kpm_options.nccl_unique_id (rank 0 calls it and
 * broadcasts the bytes to the other ranks out of band, e.g. with torch.distributed). */
kpm_status kpm_get_unique_id(void* out128);

/* Create a context on opt->device.  nranks > 1: also creates the NCCL communicator
 * (collective).  *out is NULL on failure. */
kpm_status kpm_create(kpm_ctx** out, const kpm_options* opt);

/* Store the Hermitian matrix H and the rescaling H~ = a(H - b 1), a > 0.
 * Builds the SELL-C-sigma copy on the device and, for nranks > 1, the
 * halo maps of the row distribution.  Hermiticity is checked only with
 * KPM_CHECK_HERMITIAN.  Replaces any previous matrix. */
kpm_status kpm_set_matrix(kpm_ctx* ctx, const kpm_csr* H, double a, double b);

/* Optional override of the order in which the sweep kernels visit the n = n_chunks SELL chunks
 * (a permutation of 0..n_chunks-1, host array; NULL returns to the library's own choice).  The
 * moments are unchanged up to the rounding of the eta sums (which stay deterministic).
 * Position i of the order is tile i / G of CTA i mod G (G = grid of the sweep launch, the SM
 * count times the CTAs per SM of the width's kernel; with several ranks the order is split
 * into the edge and the interior list, each keeping its relative order).
 * Without a call the library picks the order itself (DESIGN.md §7 "Chunk order"): for the
 * block-cache kernels (R = 16, 32), which reuse V blocks between a CTA's consecutive tiles, and
 * for any kernel when the matrix's storage-order neighbour window exceeds 32 MB (e.g. the
 * 400x400x40 TI at R = 32: 65 MB), the lock-step line / strip walk of kpm_plan_chunk_order derived
 * from the matrix's chunk adjacency; otherwise storage order.  Pass the identity permutation
 * to force storage order.  Reset by kpm_set_matrix. */
kpm_status kpm_set_chunk_order(kpm_ctx* ctx, const int64_t* order, int64_t n);

/* KPM-DOS moments with R random start vectors |rand()>: Z4 phases
 * {1, i, -1, -i} from Philox4x32-10 keyed by (global row, global column, seed) (DESIGN.md
 * R6), so the result does not depend on nranks or the SELL permutation.
 *   M     number of moments, even, >= 2: M/2 sweeps = init + (M/2 - 1) aug_spmmv sweeps.
 *   R     number of random vectors, >= 1 (processed in blocks of at most 32 columns).
 *   mu    out, host, M doubles: mu_n = (1/R) sum_r Re m_n^(r) with m_0 = eta_0, m_1 = eta_1,
 *         m_2k = 2 eta_2k - m_0, m_2k+1 = 2 eta_2k+1 - m_1; E[mu_n] = tr T_n(H~).
 *         Identical on all ranks.
 *   eta   out, optional (NULL), host, 2*R*M doubles: eta_n of column r at [(r*M + n)*2 + {re,im}].
 * Returns KPM_WDIVERGED (after writing mu/eta) if |mu_n| > mu_0 (1 + 1e-8) for some n. */
kpm_status kpm_moments(kpm_ctx* ctx, int M, int R, uint64_t seed, double* mu, double* eta);

/* Same with explicit start vectors: v0 = host, (row_end-row_begin) x R row-major complex
 * block of this rank's rows (2*n_loc*R doubles).  mu uses the same formula (not normalised
 * by eta_0).  KPM_EZERONORM if a column has eta_0 == 0 (mu/eta still written). */
kpm_status kpm_moments_v0(kpm_ctx* ctx, int M, int R, const double* v0, double* mu, double* eta);

/* The paper's three optimisation stages (Figs. 3-5), same outputs as
 * kpm_moments, for measuring what fusion and blocking buy:
 *   KPM_STAGE_NAIVE      Fig. 3: per column, separate spmv, axpy, scal, axpy, nrm2, dot kernels
 *                        (single rank only)
 *   KPM_STAGE_AUG_SPMV   Fig. 4: per column, the fused sweep with block width 1 ("throughput
 *                        mode" of Table III when the columns are independent runs)
 *   KPM_STAGE_AUG_SPMMV  Fig. 5: = kpm_moments (all columns in one sweep). */
enum { KPM_STAGE_NAIVE = 0, KPM_STAGE_AUG_SPMV = 1, KPM_STAGE_AUG_SPMMV = 2 };
kpm_status kpm_moments_stage(kpm_ctx* ctx, int stage, int M, int R, uint64_t seed, double* mu, double* eta);

/* The paper's bottleneck-analysis kernels (Figs. 8-9): run n_sweeps (>= 1) of one
 * kernel kind at block width R (1, 2, 4, 8, 16 or 32) on the current matrix, single rank
 * (KPM_ESTATE otherwise, or if the matrix does not fit the tiled feed):
 *   KPM_SWEEP_AUG        the fully augmented sweep of kpm_moments (dots computed, discarded),
 *   KPM_SWEEP_AUG_NODOT  the same without the on-the-fly dot products,
 *   KPM_SWEEP_SPMMV      the plain SpMMV  W = H V.
 * V = the Z4 block of kpm_moments(seed) (columns 0..R-1), W = 0 before the first sweep; every
 * sweep reads the same V (no swap), so the augmented kinds leave W = 2a(H - b)V after an odd
 * number of sweeps and 0 after an even one.
 *   ms_per_sweep  out (NULL to skip): average device time of one sweep (CUDA events).
 *   w_out         out (NULL to skip), host: the final W, n_loc x R row-major complex, local
 *                 row order (2*n_loc*R doubles). */
enum { KPM_SWEEP_AUG = 0, KPM_SWEEP_AUG_NODOT = 1, KPM_SWEEP_SPMMV = 2 };
kpm_status kpm_sweep_kernel(kpm_ctx* ctx, int kind, int R, uint64_t seed, int n_sweeps, double* ms_per_sweep,
                            double* w_out);

/* Device time of the last kpm_moments* call, measured with CUDA events on the context's
 * stream: total_ms = start-vector init .. last eta reduction; sweep_ms = average duration
 * of one main aug_spmmv sweep (the hot kernel); n_sweeps = main sweeps timed. */
kpm_status kpm_last_timing(const kpm_ctx* ctx, double* total_ms, double* sweep_ms, int* n_sweeps);

/* KPM_TIMING only: the device time (ms, CUDA events on the context's stream) of every sweep of
 * the last kpm_moments* call, in order (per column block of 32: the init sweep, then the M/2 - 1
 * main sweeps).  ms = NULL: *n = the number available; otherwise *n is the capacity on entry and
 * the number written on return.  Without KPM_TIMING, *n = 0. */
kpm_status kpm_last_sweep_times(const kpm_ctx* ctx, double* ms, int64_t* n);

/* Name of the aug_spmmv kernel variant the last kpm_moments* call ran (feed, lanes per row,
 * unroll), e.g. "staged.lpr16.u4".  "" before the first call.  The
 * environment variable KPM_VARIANT=<i> (read by kpm_create) selects variant i of a block
 * width for tuning; the default is variant 0. */
const char* kpm_last_kernel(const kpm_ctx* ctx);

/* Name of kernel variant `variant` (the KPM_VARIANT index) of block width R (1, 2, 4, ..., 32),
 * NULL if there is none; host-only, needs no GPU.  Variant 0 is the width's default. */
const char* kpm_variant_name(int R, int variant);

/* Sizes of the SELL copy, for kpm_export_sell.  n_chunks*C = n_pad. */
typedef struct {
  int64_t n_loc;     /* local rows                                       */
  int64_t n_pad;     /* n_chunks * C                                     */
  int64_t n_chunks;
  int64_t n_slots;   /* cptr[n_chunks]: stored entries including padding */
  int64_t n_halo;    /* halo rows appended after n_pad                   */
  int C, sigma;
} kpm_sell_info;

kpm_status kpm_get_sell_info(const kpm_ctx* ctx, kpm_sell_info* info);

/* Copy the SELL arrays to host buffers sized from kpm_sell_info:
 * val 2*n_slots doubles, col n_slots int32, cptr n_chunks+1 int64, perm n_loc int32
 * (perm[p] = local row stored at position p), halo n_halo int64 (global column of each
 * halo slot).  Any pointer may be NULL to skip that array. */
kpm_status kpm_export_sell(const kpm_ctx* ctx, double* val, int32_t* col, int64_t* cptr,
                           int32_t* perm, int64_t* halo);

/* The halo exchange plan of this rank (nranks > 1; zero runs on one rank), as kpm_set_matrix
 * built it (SURVEY §8(b) kpm_export_halo; the halo slot ids themselves: kpm_export_sell `halo`).
 *   recv: 4 int64 per run (owner rank, first global row, count, first halo slot): halo slots
 *         [slot, slot + count) receive the owner's global rows [first, first + count).
 *   send: 4 int64 per run (destination rank, first local position, count, first halo slot in
 *         the destination's vectors): after every sweep these rows of the new W go there.
 * recv / send = NULL: only the counts; otherwise *n_recv / *n_send are the capacities (runs),
 * KPM_EINVAL if too small.  Both counts are set on return. */
kpm_status kpm_export_halo(const kpm_ctx* ctx, int64_t* n_recv, int64_t* recv, int64_t* n_send, int64_t* send);

/* Host-only planning of the halo exchange (no GPU needed; the same code kpm_set_matrix
 * runs).  Row distribution: rank q owns global rows [row_begins[q], row_begins[q+1]).
 * kpm_plan_recv: this rank's receive runs, from its CSR rows (row_ptr, global col) --
 *   4 int64 per run: (owner rank, first global row, count, first halo slot).  Halo slots are
 *   the distinct remote columns ordered by (owner, global id).  Call with runs = NULL to get
 *   *n_runs; otherwise *n_runs is the capacity in runs.
 * kpm_plan_send: the send runs answering the n_req (first global row, count) pairs `req`
 *   that rank `peer` requested from this rank (rows [row_begin, row_end), sigma = 1) --
 *   3 int64 per run: (peer, first local position, count).  KPM_ERANGE if a request is not
 *   inside this rank's rows. */
kpm_status kpm_plan_recv(int nranks, const int64_t* row_begins, int rank, const int64_t* row_ptr,
                         const int64_t* col, int64_t* n_runs, int64_t* runs);
kpm_status kpm_plan_send(int64_t row_begin, int64_t row_end, int peer, int64_t n_req, const int64_t* req,
                         int64_t* n_runs, int64_t* runs);

/* Host-only: the library's default chunk order (the locality walk kpm_moments uses when no
 * kpm_set_chunk_order is given; DESIGN.md §7 "Chunk order").  nbr_ptr (n_chunks+1) / nbr: for
 * every chunk the chunks all of whose C rows it reads (block neighbours, CSR layout, ids in
 * [0, n_chunks)); grid: CTAs of the sweep launch (lines per round); width: 1 = single lines, 2 =
 * strips of two adjacent lines walked step by step; skip (NULL or n_chunks flags): chunks left out
 * of the lines and put last (the edge chunks of a multi-rank split).  order: out, n_chunks int64,
 * a permutation.  KPM_ERANGE for a neighbour id out of range. */
kpm_status kpm_plan_chunk_order(int64_t n_chunks, const int64_t* nbr_ptr, const int64_t* nbr, int64_t grid,
                                int width, const int8_t* skip, int64_t* order);

/* Density of states from the moments (north_star item 5; Eq. (2) `DOS`; the
 * "second computationally inexpensive step" of P:258-260).  Host only, no context.
 *   mu        M moments mu_n = tr T_n(H~) as returned by kpm_moments (mu_0 = N).
 *   a, b      the rescaling H~ = a(H - b), a > 0.
 *   energies  K energies of H (host), or NULL for the K Chebyshev nodes x_k = cos(pi(k+1/2)/K)
 *             mapped to E = x/a + b.
 *   kernel    KPM_KERNEL_JACKSON (damping g_n of the KPM review [Weisse06] cited at P:78) or
 *             KPM_KERNEL_NONE (g_n = 1).
 *   E_out, rho_out  K doubles each: rho(E) = a [g_0 mu_0 + 2 sum g_n mu_n T_n(x)] / (pi sqrt(1-x^2)),
 *             x = a(E - b); 0 where |x| >= 1.  Integrates to mu_0 = N. */
enum { KPM_KERNEL_NONE = 0, KPM_KERNEL_JACKSON = 1 };
kpm_status kpm_dos(int M, const double* mu, double a, double b, int K, const double* energies, int kernel,
                   double* E_out, double* rho_out);

/* Human-readable description of the last error on ctx (or of the last kpm_create failure
 * when ctx is NULL).  Valid until the next call on ctx. */
const char* kpm_last_error(const kpm_ctx* ctx);

/* Release everything.  NULL-safe. */
void kpm_destroy(kpm_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* KPM_H */

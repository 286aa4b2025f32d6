/*
 * appd.h -- C ABI of libappd, the B200 (sm_100a) all-points minimax path
 * distance (APPD) library.
 *
 * The operation (arxiv 2407.07058, PAPER.md):
 *   Eq. 1-2: for vertices i, j of an undirected weighted graph G,
 *     M(i,j | G) = min over all paths p from i to j of max_weight(p).
 *   the APPD is the n x n matrix of M(i,j); "a dataset X can be
 *     straightforwardly converted to a complete graph" (points mode; the edge
 *     weight is the Euclidean distance, reading Q6, computed by the
 *     pinned fp32 formula R1: acc=+0; for k<d: t=fl(x_ik-x_jk); acc=fmaf(t,t,acc);
 *     w=sqrtf(acc)).
 *   P:L93-98 (Algorithm 4): the APPD follows from a minimum spanning tree: its
 *     edges removed from large to small split the vertex set, and every pair
 *     across a split gets the removed edge's weight.  libappd computes the same
 *     matrix with an MST stage (Boruvka), an edge sort and a dendrogram
 *     (leaf order pi, merge heights h) and a fill that writes
 *     M[pi_a][pi_b] = max(h[a..b-1]).
 *   P:L50, P:L119 (widest path): sense = -1 computes the widest-path APPD
 *     (maximum spanning tree, minimum over the path) -- weights mode, and points
 *     mode on the exact FP32 engine or the Prim variant (the tensor-core filter
 *     finds minimum edges only).
 *
 * Conventions for every call:
 *   - Matrices are fp32, row-major, contiguous, leading dimension n (W, M) or
 *     d (X).  Indices are 0-based.
 *   - M[i][i] = +0.0 (the empty path, reading Q3).  Every other entry
 *     is bit-identical to one input weight (weights mode) or one R1 weight
 *     (points mode).  -0.0 input weights are read as +0.0 (reading Q5).
 *   - Unless a name ends in _host, pointers are CUDA device pointers on the
 *     context's device; host pointers are rejected with
 *     APPD_ERR_INVALID_ARGUMENT.  The caller owns every buffer it passes.
 *   - Calls enqueue work on the context's stream and return after it has
 *     completed (so data-dependent validation errors can be reported).
 *     Ordering against work on OTHER streams is the caller's: the
 *     library-owned stream (cuda_stream NULL) is a cudaStreamNonBlocking
 *     stream, unordered with the legacy default stream, so inputs produced
 *     on another stream must be complete (or that stream passed through
 *     appd_set_stream) before the call.  The Python binding passes the
 *     caller's torch.cuda.current_stream(device) on every call.
 *   - Every call returns a status; nothing throws across the ABI.  After a
 *     CUDA or NCCL failure the context is poisoned: later calls return
 *     APPD_ERR_POISONED and only appd_destroy is valid.
 *   - A context is not thread-safe: use one host thread per context.
 *   - Multi-GPU (world > 1): one process per GPU, every rank calls the solve
 *     with the same n (and d).  Rank r owns the rows [row0, row0+rows) of M
 *     returned by appd_row_range, and M points to that rows x n block.  Points
 *     mode: X is replicated on every rank.  Weights mode: W points to the
 *     rank's rows x n row block; symmetry is checked inside the rank's diagonal
 *     block only.  Every solve starts with an agreement collective over (entry
 *     point, n, d, the options that steer the control flow, and in points mode a
 *     position-keyed 64-bit checksum of X): if any rank differs, every rank
 *     returns APPD_ERR_INVALID_ARGUMENT instead of hanging in a later collective.
 *   - Validation reports one offender: the first non-finite value in row-major
 *     order if there is any, else the first nonzero diagonal entry, else the
 *     first asymmetric pair (i, j) with i < j in row-major order.
 */
#ifndef APPD_H
#define APPD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct appd_ctx appd_ctx; /* opaque: device, stream, workspace, optional NCCL communicator */

typedef enum {
  APPD_OK = 0,
  APPD_ERR_INVALID_ARGUMENT = 1, /* n < 1, d < 1, NULL or host pointer, bad option */
  APPD_ERR_NONFINITE = 2,        /* NaN or +-Inf in W or X; appd_error_index gives (i, j) */
  APPD_ERR_NOT_SYMMETRIC = 3,    /* W[i][j] != W[j][i] bitwise (after -0 -> +0); first (i, j), i < j */
  APPD_ERR_BAD_DIAGONAL = 4,     /* W[i][i] is not +-0; (i, i) */
  APPD_ERR_UNSUPPORTED = 5,      /* size beyond the supported index widths, or option not built */
  APPD_ERR_OUT_OF_MEMORY = 6,    /* device or pinned host allocation failed */
  APPD_ERR_CUDA = 7,             /* CUDA runtime error (context poisoned) */
  APPD_ERR_NCCL = 8,             /* NCCL error (context poisoned) */
  APPD_ERR_POISONED = 9          /* an earlier call failed with CUDA/NCCL error */
} appd_status;

/* MST variant (appd_options.variant) */
#define APPD_VARIANT_AUTO 0
#define APPD_VARIANT_PRIM 1    /* Prim's n - 1 sequential steps in ONE persistent
                                  CTA with the input in shared memory; it emits the leaf order and merge
                                  heights directly (no edge sort, no dendrogram build) and validates the
                                  input in the same launch.  Fits weights n <= 300 and points with
                                  n * (d + 3) <= ~56K words and n <= 2048; needs the whole input (not with
                                  sharded weights, the streamed output or fp64): otherwise a solve returns
                                  APPD_ERR_UNSUPPORTED.  Points with world > 1 run it on every rank. */
#define APPD_VARIANT_BORUVKA 2 /* row-parallel Boruvka rounds (any n, shards over ranks) */
/* APPD_VARIANT_AUTO takes Prim where it fits and is faster by measurement (weights n <= 300;
 * points n <= 1024 with n * (d + 8) <= 20480, default engine; profiles/r02/crossover.txt),
 * else Boruvka. */

typedef struct {
  uint32_t struct_size;          /* = sizeof(appd_options); set by appd_options_init */
  int32_t device;                /* CUDA device ordinal (default 0) */
  void* cuda_stream;             /* cudaStream_t to run on; NULL = library-owned stream */
  int32_t rank, world;           /* process rank / count (default 0 / 1) */
  const uint8_t* nccl_unique_id; /* world > 1: 128-byte ncclUniqueId from appd_get_nccl_unique_id on rank 0 */
  int32_t variant;               /* APPD_VARIANT_* (default AUTO) */
  int32_t validate;              /* 1 = check W/X (default), 0 = trust the input */
  int32_t sense;                 /* +1 minimax (default), -1 widest path (points: exact engine / Prim) */
  int32_t timing;                /* 1 = record per-stage CUDA events (appd_get_stats: ms_validate .. ms_total,
                                    ms_tcscan), 2 = also per-round scan events (ms_scan; each event costs
                                    a few us of stream time), default 0 */
  int32_t dendrogram;            /* 0 auto, 1 host union-find, 2 GPU */
  int32_t points_engine;         /* points-mode MST scan: 0 auto, 1 exact FP32 (CUDA cores), 2 tensor-core
                                    filter + exact recheck of the survivors (tcgen05) */
  int32_t topk;                  /* tensor-core engine: per-row candidate cache length K built in round 0
                                    (0 = auto (8), 4/8/16/32; -1 = no cache: every round scans all rows) */
  int32_t finish_k;              /* tensor-core engine: finish the MST on the contracted component graph
                                    once at most this many components remain (0 = auto (128), -1 = never;
                                    at most 128) */
  int32_t metric;                /* points mode (NEXT-3): 0 Euclidean R1 (default), 1 Manhattan (L1: fp32
                                    sum of |x_k - y_k| in k order), 2 Chebyshev (L-inf: max |x_k - y_k|);
                                    L1 / L-inf run the exact FP32 engine (the tensor-core filter is
                                    Euclidean) and the MST on the distance itself */
  /* world > 1: exchange backend.  NULL (default): NCCL over NVLink, communicator built
   * from nccl_unique_id.  Non-NULL: every collective of the solve (the solve-start
   * agreement, the validation verdict, the per-round all-reduce(min) of per-component edge
   * keys, the component-matrix all-reduce) is copied to host memory and handed to this
   * callback, which must all-reduce `count` uint64 words in place over the `world` ranks
   * (op APPD_REDUCE_MIN or APPD_REDUCE_MAX, unsigned order) and return 0; any other value
   * makes the call fail with APPD_ERR_NCCL (context poisoned).  For MPI / gloo users and
   * the multi-process tests; results are identical to the NCCL backend.
   * world 1 with nccl_unique_id or host_allreduce set: the solve takes the same
   * multi-rank path over a one-rank communicator (every exchange still issued), so the
   * transport can be checked on one GPU; results equal the plain world-1 solve's. */
  int32_t (*host_allreduce)(void* user, uint64_t* words, int64_t count, int32_t op);
  void* host_allreduce_user;
  int32_t timeout_ms;            /* world > 1, NCCL backend: deadline of every wait on work that
                                    contains a collective (0 = 300000 ms).  Past it, or when
                                    ncclCommGetAsyncError reports an error, the communicator is
                                    aborted and the call returns APPD_ERR_NCCL (poisoned) instead
                                    of hanging on a dead or diverged peer */
  int32_t list_cap;              /* tensor-core engine: capacity (entries) of the round-0 candidate
                                    list, 0 = auto (32 n + 65536).  Rows whose candidates do not fit
                                    are answered exactly by a full-row scan, so a small value only
                                    slows the solve (used by the tests to force that path) */
  int32_t wide_keys;             /* points: 1 = the wide-key exact engine (two-step component reduction,
                                    automatic above n = 131072) at any n -- the tests check it there
                                    against the oracle; 0 (default) = automatic */
  int32_t reserved[3];
} appd_options;

/* op argument of appd_options.host_allreduce */
#define APPD_REDUCE_MIN 0
#define APPD_REDUCE_MAX 1

typedef struct {
  uint32_t struct_size; /* = sizeof(appd_stats) */
  int32_t variant;      /* variant used by the last solve */
  int32_t rounds;       /* Boruvka rounds (0 for Prim) */
  int32_t dendrogram;   /* 1 host, 2 GPU, 0 none (Prim) */
  int64_t n, d, row0, rows;
  /* per-stage device time of the last solve in ms (timing = 1), else 0 */
  double ms_validate, ms_mst, ms_sort, ms_dendrogram, ms_prep, ms_fill, ms_total;
  int64_t kernel_launches; /* kernels launched by the last solve */
  int64_t fill_launches;   /* launches of the fill kernel in the last solve */
  int64_t fill_bytes;      /* bytes the fill wrote (algorithmic: rows * n * 4) */
  int64_t tc_candidates;   /* points mode, tensor-core engine: survivors re-checked exactly (all rounds) */
  int32_t points_engine;   /* engine used: 1 exact, 2 tensor core */
  int32_t exact_rounds;    /* rounds that ran the exact scan (engine 1, or a candidate-buffer overflow) */
  double ms_scan;          /* device time of the MST scan kernels (timing = 1) */
  int64_t scan_launches;   /* launches of the MST scan kernels */
  int64_t tc_fallback_rows; /* tensor-core engine: rows re-scanned exactly over all columns (all rounds) */
  double ms_tcscan;         /* tensor-core scan kernel time summed over rounds (timing = 1) */
  int64_t tcscan_launches;  /* launches of the tensor-core scan kernel */
  double tcscan_flops;      /* algorithmic flops of those launches: 2 * rows * n * d per round (the Gram term) */
  int32_t topk;             /* cache length K used (0: no cache) */
  int32_t rescan_rounds;    /* rounds >= 1 that needed a tensor-core re-scan */
  int64_t cache_invalid_rows; /* rows whose round-0 candidate list overflowed (always re-scanned) */
  int64_t rescan_rows;      /* rows re-scanned in rounds >= 1 (summed over rounds) */
  int64_t rescan_blocks;    /* 512-row blocks re-scanned in rounds >= 1 (summed over rounds) */
  int32_t cm_k;             /* components left when the component-matrix finish ran (0: not used) */
  int32_t cm_retries;       /* solves repeated without the component matrix (its candidate list overflowed) */
  int64_t collectives;      /* world > 1: all-reduces issued by the last solve (agreement, verdict, rounds) */
} appd_stats;

/* Fill *opt with defaults (device 0, own stream, world 1, AUTO, validate, minimax). */
void appd_options_init(appd_options* opt);

/* Create a context.  opt may be NULL (defaults).  world > 1 initialises NCCL
 * (collective over the ranks).  On failure *out is NULL. */
appd_status appd_create(appd_ctx** out, const appd_options* opt);

/* Set the stream later calls run on (NULL = library-owned stream). */
appd_status appd_set_stream(appd_ctx* ctx, void* cuda_stream);

/* Weights mode.  W: n x n (world 1) or this rank's rows x n block; M: rows x n.
 * Validation (validate = 1): finite, W[i][i] == +-0, W[i][j] == W[j][i]. */
appd_status appd_solve_weights(appd_ctx* ctx, const float* W, int64_t n, float* M);

/* Points mode.  X: n x d (replicated on every rank); M: rows x n.  W is never
 * materialised.  n <= 131072 packs (bits(d^2), pair index) into one 64-bit key (tensor-core
 * engine); 131072 < n <= 2^20 uses wide keys on the exact engine (see appd_solve_points_sink). */
appd_status appd_solve_points(appd_ctx* ctx, const float* X, int64_t n, int64_t d, float* M);

/* The same with HOST buffers (pinned or pageable): copies X/W in and M out on
 * the context stream, inside the call. */
appd_status appd_solve_points_host(appd_ctx* ctx, const float* X_host, int64_t n, int64_t d, float* M_host);
appd_status appd_solve_weights_host(appd_ctx* ctx, const float* W_host, int64_t n, float* M_host);

/* NEXT-4 ("at least O(n^2)"): points mode with the n x n output
 * streamed to HOST memory in blocks of block_rows original rows (0: ~1 GiB per block), so
 * n is bounded by host memory, not HBM.  X_host: n x d fp32 (host); M_host: n x n fp32
 * host buffer (pinned for full PCIe overlap; pageable works, slower).  The MST and the
 * dendrogram run once; each block's rows are filled into one of two device buffers while
 * the previous block is copied out on a second stream.  Same results, validation and
 * errors as appd_solve_points; one rank only; the device holds X, the O(n) state and
 * 2 x block_rows x n floats. */
appd_status appd_solve_points_stream(appd_ctx* ctx, const float* X_host, int64_t n, int64_t d, float* M_host,
                                     int64_t block_rows);

/* NEXT-4, outputs beyond host memory too: as appd_solve_points_stream, but each block of
 * block_rows rows (0: ~1 GiB) is handed to sink(user, row0, rows, block) in row order once
 * its copy to a pinned staging buffer is complete -- block is rows x n fp32 row-major, valid
 * only during the call -- while the GPU fills and copies the next block.  A non-zero return
 * stops the solve with APPD_ERR_INVALID_ARGUMENT.  Points mode up to n = 2^20: above
 * n = 131072 the 64-bit (weight, pair index) edge key does not fit, and the MST runs on
 * the exact FP32 engine with a two-step component reduction (minimum weight, then minimum
 * pair index among the ties; SURVEY §8(a) key note).  One rank only. */
appd_status appd_solve_points_sink(appd_ctx* ctx, const float* X_host, int64_t n, int64_t d, int64_t block_rows,
                                   int32_t (*sink)(void* user, int64_t row0, int64_t rows, const float* block),
                                   void* user);

/* NEXT-3 ("float64" weights): appd_solve_weights on an fp64 weight
 * matrix.  W: DEVICE n x n fp64 row-major; M: DEVICE n x n fp64, distinct from W.  The
 * method only compares and copies weights, so every M entry is bit-identical to
 * a W entry (or +0 on the diagonal) and to the fp64 oracle.  Same validation (finite, +-0
 * diagonal, symmetric after -0 -> +0; first offender by row-major index) and errors as
 * appd_solve_weights; opt.sense -1 gives the widest-path APPD.  One rank only (world > 1:
 * APPD_ERR_UNSUPPORTED); no candidate cache (every round rescans W); n <= 92682.
 * appd_last_dendrogram is not available after this call (APPD_ERR_INVALID_ARGUMENT). */
appd_status appd_solve_weights_f64(appd_ctx* ctx, const double* W, int64_t n, double* M);

/* NEXT-2: the paper's comparison algorithm, the minimax variant of
 * Floyd–Warshall ("a modified version of the Floyd-Warshall algorithm", Fig. floyd
 * k outermost, M[i][j] = min(M[i][j], max(M[i][k], M[k][j])); O(n^3)),
 * as a blocked (min, max) closure on the GPU.  W, M: DEVICE n x n fp32 row-major, distinct
 * buffers (M is overwritten; W is read only).  Same validation and error behaviour as
 * appd_solve_weights; opt.sense -1 gives the widest-path APPD.  -0 reads as +0 and the
 * diagonal is +0 (Q3, Q5), so M is bit-identical to appd_solve_weights' result.  One
 * rank only (world > 1: APPD_ERR_UNSUPPORTED); n <= 65536. */
appd_status appd_floyd_weights(appd_ctx* ctx, const float* W, int64_t n, float* M);

void appd_destroy(appd_ctx* ctx); /* NULL-safe; frees the workspace and the NCCL communicator */

/* ---- support ---- */

/* Rows of M this rank owns: [row0, row0 + rows) (host-only; no device needed). */
appd_status appd_row_range(const appd_ctx* ctx, int64_t n, int64_t* row0, int64_t* rows);
/* Same without a context: the row split rank r of world uses. */
appd_status appd_row_range_of(int64_t n, int32_t rank, int32_t world, int64_t* row0, int64_t* rows);

/* R1 weights for rows [row0, row0+rows) of the complete graph of X (device, rows x n). */
appd_status appd_points_weights(appd_ctx* ctx, const float* X, int64_t n, int64_t d, int64_t row0, int64_t rows,
                                float* Wblock);

/* Test hook for the tensor-core engine: the raw fp32 accumulator of the first
 * 512 (padded) rows against all columns (tc_out, 512 x npad, npad = n rounded up
 * to a multiple of 512) and a plain FP32 dot product of the same packed fp16
 * operands (ref_out, same shape).  Device pointers. */
appd_status appd_debug_tc_gram(appd_ctx* ctx, const float* X, int64_t n, int64_t d, float* tc_out, float* ref_out);

/* 128-byte ncclUniqueId for appd_options.nccl_unique_id (call on rank 0 only). */
appd_status appd_get_nccl_unique_id(uint8_t out[128]);

/* Statistics of the last solve; stats->struct_size must be sizeof(appd_stats). */
appd_status appd_get_stats(const appd_ctx* ctx, appd_stats* stats);

/* Test hook: leaf order pi (int32[n]) and merge heights h (float[n-1]) of the last
 * solve, to host memory.  Either pointer may be NULL. */
appd_status appd_last_dendrogram(const appd_ctx* ctx, int32_t* pi_host, float* h_host, int64_t n);

/* Offending indices of the last NONFINITE / NOT_SYMMETRIC / BAD_DIAGONAL status. */
appd_status appd_error_index(const appd_ctx* ctx, int64_t* i, int64_t* j);

const char* appd_last_error(const appd_ctx* ctx); /* message of the last failure ("" if none) */
const char* appd_status_string(appd_status s);

/* Library build identification: "libappd <version> sm_100a". */
const char* appd_version(void);

#ifdef __cplusplus
}
#endif

#endif /* APPD_H */

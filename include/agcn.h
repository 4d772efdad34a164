/*
 * agcn.h -- C ABI of the B200-native (sm_100a) Accel-GCN aggregation SpMM, Y = A.X.
 *
 * The method is arXiv 2308.11825 (Accel-GCN).  P:n below is /root/reference/PAPER.md line n.
 *   - GCN feature aggregation X^{l+1} = sigma(A' Y^l) is an SpMM of a sparse adjacency
 *     with a dense feature matrix.  This library computes the SpMM (no sigma).
 *   - agcn_plan builds the preprocessing of section III-C: degree sorting, the
 *     partition patterns of Algorithm 1 and the block-level partition of
 *     Algorithm 2, packed as one 128-bit descriptor per block.
 *   - agcn_spmm runs the SpMM over that metadata with the combined-warp mapping of the
 *     dense column dimension and hierarchical accumulation.
 *
 * Conventions for every entry point:
 *   - Indices are int32, values fp32.  Dense matrices are row-major with ld = F.
 *   - "DEVICE" pointers are CUDA device pointers on the current device; "HOST" pointers
 *     are host memory (pinned recommended).  No call takes ownership of caller memory.
 *   - Errors are reported by return code only (never abort/exit/throw across the ABI);
 *     functions returning a plan return NULL on failure.  agcn_last_status() and
 *     agcn_last_error() give the code and a message for the calling thread.
 *   - Streams are cudaStream_t (agcn_stream_t is the same type); NULL = legacy default.
 */
#ifndef AGCN_H
#define AGCN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

struct CUstream_st;
typedef struct CUstream_st* agcn_stream_t; /* == cudaStream_t */

typedef struct agcn_plan_s* agcn_plan_t;   /* opaque, immutable after creation */

typedef enum {
    AGCN_OK = 0,
    AGCN_ERR_INVALID_ARG = 1, /* null pointer, negative size, nnz >= 2^31, F <= 0, X == Y ... */
    AGCN_ERR_BAD_CSR = 2,     /* rowptr not monotone, rowptr[n]-rowptr[0] != nnz, colidx out of range */
    AGCN_ERR_OOM = 3,         /* device allocation failed */
    AGCN_ERR_CUDA = 4,        /* any other CUDA runtime error (message has the CUDA string) */
    AGCN_ERR_OVERFLOW = 5,    /* a descriptor field does not fit (16-bit info halves, 32-bit loc) */
    AGCN_ERR_UNSUPPORTED = 6  /* configuration outside this build's limits (see agcn_plan_ex) */
} agcn_status_t;

typedef enum {
    AGCN_PARTITION_BLOCK = 0, /* degree sort + block-level partition (the method) */
    AGCN_PARTITION_WARP = 1   /* warp-level partition, no sort (ablation arm, Fig. 3(b)) */
} agcn_partition_t;

typedef struct {
    int32_t max_block_warps;   /* Alg. 1 max_block_warps; default 12 */
    int32_t max_warp_nzs;      /* Alg. 1 max_warp_nzs; default 32.
                                  Both 0: chosen from n and nnz (measured rule, DESIGN.md 9;
                                  agcn_plan_stats reports the values used) */
    int32_t partition;         /* agcn_partition_t; default AGCN_PARTITION_BLOCK */
    int32_t validate;          /* 1 (default): check the CSR on device -> AGCN_ERR_BAD_CSR */
    int64_t n_cols;            /* columns of A (rows of X); 0 -> n */
    agcn_stream_t stream;      /* stream the plan is built on; default NULL */
    /* Optional column relabel for a padded all-gather layout (multi-GPU):
       if col_nparts > 0, column j is stored as p*col_slot_rows + (j - col_bounds[p]) where
       col_bounds[p] <= j < col_bounds[p+1] (HOST array of col_nparts+1 int64).  The plan's
       SpMM then reads X in that padded layout (col_nparts * col_slot_rows rows). */
    const int64_t* col_bounds;
    int32_t col_nparts;
    int64_t col_slot_rows;
    /* Hot X rows (north_star: "an L2 access-policy window keeping hot X rows resident"): the
       plan marks the hot_rows highest-degree vertices -- the tail of the degree order it has
       just computed -- as hot, and agcn_spmm gathers their X rows into a compact
       plan-owned buffer that an L2 persisting window (or evict_last hints) keeps resident.
       Row degree stands in for column in-degree (correlation 0.997-0.9997 on the power-law
       configs, profiles/r02_c5_roof.md).  Needs a square A (n_cols == n) without col_bounds.
       -1 (default): auto -- min(n, 524288) when n >= 2^19 (X of 128+ MiB at F = 64), else 0;
       0: off; > 0: that many rows (capped at the rows of degree >= 1).  Results do not depend
       on it.  Costs the plan one lookup per nonzero (C5: +0.4 ms). */
    int64_t hot_rows;
    int32_t small_plan;        /* 1 (default): graphs within the one-CTA limits (see agcn_plan_ex)
                                  take the one-CTA plan; 0: always the general plan (same
                                  metadata; for tests and measurements) */
    int32_t chunk_buckets;     /* oversized-chunk execution order (agcn_spmm_opts_t.chunk_order):
                                  buckets of in-row position; 0 (default): 64 */
} agcn_opts_t;

typedef struct {
    int64_t n, n_cols, nnz;
    int64_t nblocks;            /* block descriptors (AGCN_PARTITION_BLOCK) */
    int64_t ntasks;             /* warp tasks (AGCN_PARTITION_WARP) */
    int64_t deg_bound;          /* max_block_warps * max_warp_nzs (Alg. 1 line 1) */
    int64_t max_deg;
    int64_t n_zero_rows;        /* degree-0 rows (sorted first, no descriptor) */
    int64_t n_oversized_rows;   /* rows with degree > deg_bound */
    int64_t n_oversized_blocks; /* descriptors of those rows (chunks of <= deg_bound nnz) */
    int32_t max_block_warps, max_warp_nzs, partition, reserved;
    size_t device_bytes;        /* device memory owned by the plan */
    int64_t hot_rows;           /* hot X rows (agcn_opts_t.hot_rows as resolved) */
} agcn_plan_stats_t;

typedef enum {
    AGCN_FIELD_PERM = 0,          /* int32[n]       sorted position -> original row (sorted_to_orig) */
    AGCN_FIELD_BLOCKS = 1,        /* uint32[4*nblocks] descriptors (deg, loc, row, info), little endian */
    AGCN_FIELD_SORTED_COLIDX = 2, /* int32[nnz]     colidx in degree-sorted row order (after relabel) */
    AGCN_FIELD_ROW_SRC_OFF = 3,   /* int32[n]       rowptr[perm[k]] - rowptr[0] */
    AGCN_FIELD_TASKS = 4,         /* uint32[4*ntasks] warp tasks (row, col, len, 0) */
    AGCN_FIELD_SORTED_ROWPTR = 5, /* int32[n+1]     row pointer of the degree-sorted CSR */
    AGCN_FIELD_HOT_COLS = 6       /* int32[hot_rows] the hot vertices (agcn_opts_t.hot_rows), ascending:
                                     the columns whose X rows agcn_spmm reads from the compact buffer */
} agcn_field_t;

/* Fill *opts with the defaults above. */
void agcn_default_opts(agcn_opts_t* opts);

/*
 * Build the degree-sort + block-partition plan on the current device (Alg. 1, Alg. 2).
 *   rowptr: DEVICE int32[n+1], non-decreasing; rowptr[0] may be nonzero (a row shard of a
 *           larger CSR) -- then colidx is indexed by the rowptr values (global arrays).
 *   colidx: DEVICE int32, entries rowptr[0] .. rowptr[n]-1 are read; 0 <= colidx < n_cols.
 *   n, nnz: rows of A and rowptr[n] - rowptr[0]; 0 <= n, 0 <= nnz < 2^31.  nnz < 0 means
 *           "read it from rowptr" (one extra readback of rowptr[0] and rowptr[n]).
 * Degree order is ascending and stable (ties keep original row order); degree-0 rows come
 * first and get no descriptor.  Step (3) of P:295 reorders the CSR: the plan stores the
 * degree-sorted row pointer, per sorted row where its entries start in the caller's vals,
 * and its own copy of colidx, kept in the caller's order so that a sorted row's column indices
 * and vals are read at the same offset (hot columns re-encoded, see hot_rows).  Ownership: the
 * plan copies what it needs -- no kernel reads rowptr or colidx after return, so they may be
 * freed or changed then.  Host synchronisation: the general block plan waits for
 * two events on opts.stream (the bucket counts + rowptr flags, then the colidx range flag), never
 * for the stream: it returns while its last kernels (degree order, Alg. 1/2 descriptors) still
 * run asynchronously on opts.stream; agcn_spmm on that stream is ordered after them and
 * agcn_spmm on another stream waits for them (event).  The AGCN_PARTITION_WARP plan and block
 * plans of graphs with n <= 32768, nnz <= 2^20, deg_bound <= 512 and at most 1024 oversized rows
 * (one CTA, same metadata) read one set of flags back mid-way.
 * Limits: deg_bound = max_block_warps*max_warp_nzs <= 2048,
 * max_block_warps < 65536 and max_warp_nzs < 65536 (16-bit info halves) -> otherwise
 * AGCN_ERR_UNSUPPORTED / AGCN_ERR_OVERFLOW.  Returns NULL on error.
 */
agcn_plan_t agcn_plan(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t nnz);
agcn_plan_t agcn_plan_ex(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t nnz,
                         const agcn_opts_t* opts);

/*
 * Y = A.X with the plan's partition.
 *   vals: DEVICE fp32, indexed like colidx (the caller's ORIGINAL CSR order, rowptr values).
 *   X:    DEVICE fp32 [n_cols x F] row-major (or the padded layout if the plan relabels).
 *   Y:    DEVICE fp32 [n x F] row-major, original row order; must not overlap X.
 * Every element of Y is written (rows of degree 0 become 0).  Asynchronous on `stream`;
 * never synchronises.  Deterministic for AGCN_PARTITION_BLOCK (fixed summation order, no
 * atomics); AGCN_PARTITION_WARP uses fp32 global atomics for rows split across warps.
 * May grow a plan-owned scratch buffer (stream-ordered) the first time a larger F is used.
 * Calls on one plan must be stream-ordered (the scratch is shared).
 * Any F >= 1 is accepted; F % 4 == 0 with 16-byte aligned X and Y takes the float4 path.
 */
agcn_status_t agcn_spmm(agcn_plan_t plan, const float* vals, const float* X, int32_t F, float* Y,
                        agcn_stream_t stream);

/* SpMM kernel variants (all compute the same Y within the tolerance; AUTO picks per F). */
typedef enum {
    AGCN_KERNEL_AUTO = 0,    /* WIDE when applicable, else GENERAL */
    AGCN_KERNEL_GENERAL = 1, /* any F: float4 (F % 4 == 0, 16-B aligned X/Y) or scalar lanes;
                                shared-memory staging of each descriptor's colidx / vals */
    AGCN_KERNEL_LOOPED = 2,  /* ablation 2 of the paper (Fig. 4(a), Table II):
                                no combined warp -- GENERAL with one warp of 32 scalar lanes per
                                row that loops over the columns in strides of 32; any F */
    AGCN_KERNEL_WIDE = 3     /* F = 8 L <= 256 (any L), 32-B aligned X/Y, max_block_warps
                                <= 32: one 256-bit row slice per lane, shuffle-broadcast CSR */
} agcn_kernel_t;

typedef enum {
    AGCN_L2_AUTO = -1,
    AGCN_L2_NONE = 0,       /* plain X-row loads */
    AGCN_L2_KEEP_ALL = 1,   /* every X-row load L2::evict_last (X that fits in L2) */
    AGCN_L2_HOT_WINDOW = 2, /* the hot buffer read under an L2 access-policy window (hitProp
                               persisting) over it; raises the DEVICE-WIDE persisting-L2 limit
                               (cudaLimitPersistingL2CacheSize) to the window size the first
                               time, which shrinks L2 for all later normal accesses of the
                               process (measured: other SpMMs 10-15 % slower).  The buffer's
                               lines are discarded from L2 after the SpMM.  Plans without hot
                               rows: NONE */
    AGCN_L2_HOT_HINTS = 3   /* hot buffer loads L2::evict_last, cold loads evict_first */
} agcn_l2_hint_t;

typedef enum {
    AGCN_AGG_SUM = 0,  /* y_i = sum_j a_ij x_j (GCN aggregation) */
    AGCN_AGG_MEAN = 1  /* y_i = sum_j a_ij x_j / deg_i, 0 for deg_i = 0 (GraphSAGE-mean) */
} agcn_aggregation_t;

typedef struct {
    int32_t kernel;       /* agcn_kernel_t; default AGCN_KERNEL_AUTO */
    int32_t l2_hint;      /* X-row L2 residency (agcn_l2_hint_t; results never depend on it).
                             Plans with hot rows always read them from the compact buffer;
                             AGCN_L2_AUTO (default): HOT_HINTS for plans with hot rows, else
                             KEEP_ALL when X fits in L2 (<= 128 MiB), else NONE
                             (profiles/r02_c5_roof.md, r02z_l2_modes.txt) */
    int32_t hot_mb;       /* HOT_* modes: MiB of hot X rows kept resident (rows = hot_mb MiB /
                             (4 F), at most the plan's hot_rows); 0 (default): the device's
                             maximum persisting-L2 size */
    /* Epilogue, applied to every output row i (fused into the WIDE kernel's stores and the
       oversized-row reduction; a separate pass over Y for the other kernels):
         y_i = agg(i) + self_scale * self[i] + bias;  y_i = max(y_i, 0) if relu
       agg(i) per `aggregation`.  GIN: self = X, self_scale = 1 + eps. */
    int32_t aggregation;  /* agcn_aggregation_t; default AGCN_AGG_SUM */
    float self_scale;     /* 0 (default): no self term */
    int32_t relu;         /* 0 (default) / 1 */
    const float* self;    /* DEVICE [n x F] row-major, row i pairs with output row i; 16-byte
                             aligned; required iff self_scale != 0 */
    const float* bias;    /* DEVICE [F], 16-byte aligned, or NULL */
    /* Fused all-gather (multi-GPU): every finished output row i is also stored to
       peer_out[q] + i * F for q < npeer -- typically this rank's slot in each peer's next-layer X
       buffer, mapped into this process with agcn_ipc_open (NVLink peer stores from the SpMM's
       own epilogue instead of a separate all-gather).  DEVICE pointers, 16-byte aligned; the
       caller orders the peers' reads (e.g. a barrier after the layer). */
    float* peer_out[8];
    int32_t npeer;        /* 0 (default) .. 8 */
    /* WIDE kernel, plans with more than 16384 oversized-row chunks: the chunks run in a kernel
       of their own (k_spmm_chunks) before the other descriptors.  0 (default): auto (F >= 32:
       U 4 rows in flight per lane at 4 CTAs/SM; else off); -1: off (one kernel for every
       descriptor); 3, 4: U 4 at that many CTAs/SM; 6: U 2 at 6 CTAs/SM.  Results are bitwise
       the same. */
    int32_t chunk_shape;
    /* Execution order of the oversized-row chunks (the descriptors keep Alg. 2's order):
       0 (default): bucketed by the chunk's position in its row (concurrent warps gather from
       the same part of X: L2 reuse across hub rows); -1: descriptor order.  Same results. */
    int32_t chunk_order;
    int32_t pad0_;
    int64_t reserved[2];
} agcn_spmm_opts_t;

/* Fill *opts with the defaults above. */
void agcn_default_spmm_opts(agcn_spmm_opts_t* opts);

/*
 * agcn_spmm with an explicit kernel choice (same contract as agcn_spmm; opts may be NULL).
 * A kernel that cannot run this F / alignment / plan returns AGCN_ERR_UNSUPPORTED.
 * AGCN_PARTITION_WARP plans ignore opts.kernel (they have their own kernel).
 */
agcn_status_t agcn_spmm_ex(agcn_plan_t plan, const float* vals, const float* X, int32_t F,
                           float* Y, agcn_stream_t stream, const agcn_spmm_opts_t* opts);

/* Release the plan's device memory, stream-ordered on the plan's stream (after its own work
   and after the most recent agcn_spmm issued on another stream); never synchronises the host.
   Work on further streams must be ordered by the caller.  NULL is a no-op. */
agcn_status_t agcn_plan_destroy(agcn_plan_t plan);

/*
 * The Alg. 1 parameters agcn_plan_ex uses when opts.max_block_warps == opts.max_warp_nzs == 0:
 * a host-only rule in n, nnz and the SM count (sms <= 0: the current device's), measured on
 * B200 (profiles/r01at_auto_partition.md).  With share = nnz / (sms * 24):
 * share < 8 -> (12, 32); share < 960 -> (4, 16), (8, 16) or (8, 32) for share / 2.5 below
 * 128, below 256, at least 256; else (32, 16) if nnz < 64 n (mean degree < 64), else (8, 32).  Never fails for
 * n, nnz >= 0 and non-NULL outputs (else AGCN_ERR_INVALID_ARG).
 */
agcn_status_t agcn_auto_partition(int64_t n, int64_t nnz, int32_t sms, int32_t* max_block_warps,
                                  int32_t* max_warp_nzs);

/* Plan statistics (host struct, filled without device synchronisation). */
agcn_status_t agcn_plan_stats(agcn_plan_t plan, agcn_plan_stats_t* out);

/* Copy one plan array (agcn_field_t) to HOST memory; bytes must equal the field size
   given in agcn_field_t (else AGCN_ERR_INVALID_ARG).  Synchronous. */
agcn_status_t agcn_plan_copy(agcn_plan_t plan, int32_t field, void* host_dst, size_t bytes);

/*
 * nnz-balanced contiguous row shards for nranks GPUs (BASELINE.json north_star):
 * bounds[0] = 0, bounds[nranks] = n, bounds[p] = first row r with
 * rowptr[r] - rowptr[0] >= floor(p * nnz / nranks).  rowptr: DEVICE int32[n+1];
 * bounds_host: HOST int64[nranks+1].  Synchronises `stream`.
 */
agcn_status_t agcn_shard_bounds(const int32_t* rowptr, int64_t n, int32_t nranks,
                                int64_t* bounds_host, agcn_stream_t stream);

/*
 * End-to-end convenience on HOST buffers: copies the CSR and X to the device, builds the
 * plan, runs `layers` propagations Y_{l+1} = A.Y_l (Y_0 = X; layers > 1 needs n_cols == n),
 * and copies the last Y back to Y_host [n x F].  Device memory is stream-ordered
 * (cudaMallocAsync) and released before return.  Synchronous.  opts may be NULL.
 */
agcn_status_t agcn_propagate_host(const int32_t* rowptr_host, const int32_t* colidx_host,
                                  const float* vals_host, int64_t n, int64_t nnz,
                                  const float* X_host, int32_t F, int32_t layers, float* Y_host,
                                  const agcn_opts_t* opts);

/*
 * Pipelined executor of agcn_propagate_host jobs (the serving path): job k's host->device
 * copies run while job k-1's result is copied back, so the PCIe link carries both directions
 * at once.  Each job computes exactly what agcn_propagate_host computes (same plan, same
 * kernels, bit-identical Y): copy the CSR + X in, agcn_plan (degree sort + Alg. 1/2, P:295,
 * P:314-382), `layers` x agcn_spmm, copy Y out.
 *
 * agcn_pipe_create: `depth` (>= 1, default 2 when <= 0) device buffer sets, reused round-robin;
 *   opts as for agcn_plan_ex (NULL = defaults; opts->stream is ignored: the executor owns one
 *   copy-in, one compute and one copy-out stream on the current device).  NULL on failure.
 * agcn_pipe_submit: enqueue one job on HOST buffers (as agcn_propagate_host: rowptr[n+1],
 *   colidx / vals indexed by rowptr values, X [n_cols x F], Y [n x F]; n_cols = opts->n_cols
 *   or n).  Enqueues the job's copy-in and returns; a worker thread owned by the executor
 *   builds the plan (it waits for the inputs), enqueues the SpMMs and the copy of Y.  Blocks
 *   only while the job's buffer slot still belongs to an earlier job the worker has not
 *   enqueued yet.  Argument errors (and rowptr[n] - rowptr[0] != nnz) are returned here; errors
 *   found later (a bad CSR, a CUDA error) are returned by agcn_pipe_wait.  The caller keeps
 *   every host buffer of the job alive and unmodified, and reads Y_host only after
 *   agcn_pipe_wait.  Host buffers should be pinned (page-locked): pageable memory works but
 *   the copies then do not overlap.  A failed job leaves the executor usable.
 * agcn_pipe_wait: blocks until every submitted job has finished (Y_host written); returns the
 *   first error of the jobs since the previous wait (that job's Y_host is not written), if any.
 * agcn_pipe_destroy: waits, then frees the device buffers and streams.  NULL is a no-op.
 */
/*
 * CUDA-graph propagation: `layers` x agcn_spmm (Y_{l+1} = A.Y_l, Y_0 = X; the SpMM of P:124-126
 * with the plan's partition) captured once and replayed with one launch -- for small
 * graphs, whose layers are bound by launch latency.
 * agcn_graph_create: X DEVICE [n_cols x F]; ybuf0, ybuf1 DEVICE [n x F] (ybuf1 unused and may be
 *   NULL when layers == 1); layer l writes ybuf[l % 2], so the result is ybuf[(layers-1) % 2].
 *   Runs the layers once eagerly (synchronously; it also grows the plan's scratch), then
 *   captures them on a private stream.  The graph keeps the pointers: every launch reads X and
 *   vals and writes the ybufs at these addresses (write new features into X in place).
 *   layers > 1 needs a square A.  NULL on failure.
 * agcn_graph_launch: asynchronous on `stream` (any stream; launches on one graph must be
 *   stream-ordered, as agcn_spmm calls on one plan).  agcn_plan_destroy is ordered after the
 *   latest launch.
 * agcn_graph_destroy: frees the graph.  The plan must outlive the graph.  While a graph of a
 *   plan exists, an agcn_spmm on that plan that would grow its scratch (a larger F than any
 *   captured one) returns AGCN_ERR_UNSUPPORTED instead of moving memory under the graph.
 */
typedef struct agcn_graph_s* agcn_graph_t;
agcn_graph_t  agcn_graph_create(agcn_plan_t plan, const float* vals, const float* X, int32_t F, int32_t layers,
                                float* ybuf0, float* ybuf1);
agcn_status_t agcn_graph_launch(agcn_graph_t graph, agcn_stream_t stream);
agcn_status_t agcn_graph_destroy(agcn_graph_t graph);

typedef struct agcn_pipe_s* agcn_pipe_t;
agcn_pipe_t   agcn_pipe_create(int32_t depth, const agcn_opts_t* opts);
agcn_status_t agcn_pipe_submit(agcn_pipe_t pipe, const int32_t* rowptr_host, const int32_t* colidx_host,
                               const float* vals_host, int64_t n, int64_t nnz, const float* X_host,
                               int32_t F, int32_t layers, float* Y_host);
agcn_status_t agcn_pipe_wait(agcn_pipe_t pipe);
agcn_status_t agcn_pipe_destroy(agcn_pipe_t pipe);

/*
 * CSR of A^T on the device, for the backward pass of a GCN layer (dX = A^T . dY).  A stable
 * counting sort of the nonzeros by column (the degree sort's machinery): row j of A^T
 * lists the rows i with a_ij != 0 in increasing i.
 *   rowptr: DEVICE int32[n+1] (rowptr[0] may be nonzero: colidx is indexed by rowptr values);
 *   colidx: DEVICE int32, 0 <= colidx < n_cols (not validated here: build a plan first).
 *   rowptr_t: DEVICE int32[n_cols+1] out (starts at 0); colidx_t: DEVICE int32[nnz] out;
 *   src: DEVICE int32[nnz] out -- entry k of A^T is entry src[k] of A (rowptr-relative),
 *        so vals_t = vals[src] (agcn_gather_vals).
 * Outputs are caller-owned and must not overlap the inputs.  Asynchronous on `stream`
 * (stream-ordered scratch, no host synchronisation).
 */
agcn_status_t agcn_transpose(const int32_t* rowptr, const int32_t* colidx, int64_t n, int64_t n_cols,
                             int64_t nnz, int32_t* rowptr_t, int32_t* colidx_t, int32_t* src,
                             agcn_stream_t stream);

/* out[k] = vals[src[k]] for k < nnz (DEVICE arrays; vals indexed rowptr-relative, like src).
   Asynchronous on `stream`. */
agcn_status_t agcn_gather_vals(const float* vals, const int32_t* src, int64_t nnz, float* out,
                               agcn_stream_t stream);

/*
 * Dense Y = X . W (+ bias, ReLU) on the tcgen05 tensor cores, kind::tf32 -- the X.W of a GCN
 * layer.  TF32 precision: operands rounded to a 10-bit mantissa,
 * fp32 accumulation: |y - y_ref| <= ~2^-9 sum_k |x_k w_k|.
 *   X:  DEVICE fp32 [M x K] row-major;  Wt: DEVICE fp32 [N x K] row-major (W transposed);
 *   Y:  DEVICE fp32 [M x N] row-major;  bias: DEVICE fp32 [N] or NULL;  relu: 0 / 1.
 * K in [4, 256] with K % 4 == 0; N in {16, 32, 64, 128, 256}; 16-byte aligned pointers;
 * (K rounded up to 32) x (128 + N) x 4 bytes must fit in shared memory -> else
 * AGCN_ERR_UNSUPPORTED.  Asynchronous on `stream`.
 */
agcn_status_t agcn_gemm_xw(const float* X, int64_t M, int32_t K, const float* Wt, int32_t N, float* Y,
                           const float* bias, int32_t relu, agcn_stream_t stream);

/*
 * agcn_gemm_xw with a precision choice (the X.W of the GCN layer):
 *   AGCN_GEMM_FP32: fp32 accuracy, |y - y_ref| <= ~2^-19 sum_k |x_k w_k| + fp32 accumulation --
 *     "3xTF32" on the tcgen05 tensor cores: both operands split in shared memory into a TF32
 *     high part (low 13 mantissa bits cleared) and the exact remainder, x w accumulated as
 *     x_hi w_hi + x_lo w_hi + x_hi w_lo (three kind::tf32 MMAs per K step of 8) for
 *     N in {16, 32, 64, 128, 256} (as column slices of W when the split W^T does not fit in
 *     shared memory with the whole N); other N: a CUDA-core fp32 FFMA kernel.
 *     K in [4, 256], K % 4 == 0; N in [4, 256], N % 4 == 0.
 *   AGCN_GEMM_TF32: as agcn_gemm_xw.
 * Same pointer / alignment rules as agcn_gemm_xw; asynchronous on `stream`.
 */
typedef enum { AGCN_GEMM_FP32 = 0, AGCN_GEMM_TF32 = 1 } agcn_gemm_precision_t;
agcn_status_t agcn_gemm_xw_ex(const float* X, int64_t M, int32_t K, const float* Wt, int32_t N, float* Y,
                              const float* bias, int32_t relu, int32_t precision, agcn_stream_t stream);

/* Device buffers that other processes can map (CUDA IPC): the fused all-gather's peer X
   buffers.  agcn_device_alloc: cudaMalloc'd (exportable) bytes; agcn_ipc_export writes a
   64-byte handle of ptr (a pointer returned by agcn_device_alloc); agcn_ipc_open maps a
   handle from another process (peer access enabled lazily) and agcn_ipc_close unmaps it. */
agcn_status_t agcn_device_alloc(size_t bytes, void** ptr);
agcn_status_t agcn_device_free(void* ptr);
agcn_status_t agcn_ipc_export(const void* ptr, void* handle64);
agcn_status_t agcn_ipc_open(const void* handle64, void** ptr);
agcn_status_t agcn_ipc_close(void* ptr);

agcn_status_t agcn_last_status(void);
const char* agcn_last_error(void);

/* Number of kernels this library has launched in this process (monotone counter). */
uint64_t agcn_launch_count(void);

/* Library version string, e.g. "agcn 0.1 sm_100a". */
const char* agcn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AGCN_H */

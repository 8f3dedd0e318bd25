/*
 * tcg.h -- C ABI of the B200-native pruned color-coding DP ("treecount-b200").
 *
 * This is the drop-in boundary for the reference's vectorized engine
 * (/root/reference/proj/include/treecount/engines.hpp:302-307 run_iteration,
 * estimator.hpp:49-93 estimate).  Plain pointers and sizes only; no
 * exceptions cross the ABI.  Status codes mirror the reference's exception
 * classes:
 *   TCG_OK        0  success
 *   TCG_EINVAL    1  std::invalid_argument (k out of range, iterations < 1,
 *                    coloring size / value mismatch, NULL arguments)
 *   TCG_ERESOURCE 2  memory_budget_error (engines.hpp:37-44) or device OOM --
 *                    the CLI's exit code 2 class (treecount_cli.cpp:501-503)
 *   TCG_ECUDA     3  CUDA failure
 *   TCG_ENONFINITE 4 non-finite rooted total (overflow guard, SURVEY finding 2)
 *   TCG_ELOGIC    5  std::logic_error (liveness / internal invariant)
 *   TCG_EPARSE    6  treecount::parse_error (graph.hpp:18-21): bad graph input
 *                    (vertex id out of range, CSR invariants) or template input
 *                    (not a tree, root out of range; templates.hpp:37-88)
 * The message of the last failure is available from tcg_last_error().
 *
 * Numerics: count tables are fp32 (SpMM neighbour sums accumulate in fp64,
 * the root and every total in fp64).  A non-root table entry is a colourful
 * sub-template count rooted at one vertex and must stay below FLT_MAX
 * (3.4e38): at the BASELINE configs the largest non-root entries are ~1e29
 * (cfg3) to ~1e34 (cfg4 bound); a graph/template whose
 * intermediate counts overflow fp32 yields an inf/nan rooted total, reported
 * as TCG_ENONFINITE -- never a silently wrong count.
 * Ownership: inputs are caller-owned and copied; outputs are caller-allocated.
 * A context is single-threaded and blocks until results are on the host.
 */
#ifndef TCG_H
#define TCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TCG_OK = 0,
  TCG_EINVAL = 1,
  TCG_ERESOURCE = 2,
  TCG_ECUDA = 3,
  TCG_ENONFINITE = 4,
  TCG_ELOGIC = 5,
  TCG_EPARSE = 6
};

#define TCG_MAX_K 20                   /* color_index.hpp:15 kMaxTemplateSize */
#define TCG_MAX_NODES (2 * TCG_MAX_K - 1)

/* Message of the most recent failure on this thread (any entry point). */
const char* tcg_last_error(void);
/* Library build string (arch, version). */
const char* tcg_version(void);

/* ------------------------------------------------------------------------
 * Host graph: symmetric CSR (== treecount::Graph::csc_col_ptr / csc_rows,
 * graph.hpp:27-42): int64 row_ptr[n+1], int32 col[nnz], rows sorted,
 * deduplicated, no self-loops.
 * ---------------------------------------------------------------------- */
typedef struct tcg_graph tcg_graph;

/* graph.hpp:65-95 from_edges: symmetrize by union, drop self-loops, dedup,
 * sort.  edges = m (u,v) int32 pairs; n_hint < 0 -> max id + 1.  Built by a
 * multithreaded radix sort on the host. */
int tcg_graph_from_edges(const int32_t* edges, int64_t m, int32_t n_hint, tcg_graph** out);
/* Adopt an existing CSR (validated: symmetric, sorted, no loops/duplicates). */
int tcg_graph_from_csr(int32_t n, const int64_t* row_ptr, const int32_t* col, tcg_graph** out);
/* synthgen.hpp:40-74 generate_rmat / 76-85 generate_erdos_renyi, bit-identical
 * edge streams (std::mt19937_64 + Rng::unit).  Harness input generators. */
int tcg_generate_rmat(int scale, int64_t edges, double a, double b, double c, double d,
                      uint64_t seed, tcg_graph** out);
int tcg_generate_erdos_renyi(int32_t n, double p, uint64_t seed, tcg_graph** out);
int tcg_graph_info(const tcg_graph* g, int32_t* n, int64_t* m, int64_t* nnz,
                   int32_t* max_degree);
/* Zero-copy views of the host CSR (valid until tcg_graph_destroy). */
const int64_t* tcg_graph_row_ptr(const tcg_graph* g);
const int32_t* tcg_graph_col(const tcg_graph* g);
void tcg_graph_destroy(tcg_graph* g);

/* ------------------------------------------------------------------------
 * Host template pieces (templates.hpp, color_index.hpp), exposed for tests
 * and plan inspection.  edges = k-1 (u,v) pairs; root < 0 = default root
 * (max-degree vertex, smallest id; templates.hpp:67-74).
 * ---------------------------------------------------------------------- */
typedef struct {
  int k, root, num_nodes;
  int size[TCG_MAX_NODES];
  int node_root[TCG_MAX_NODES];
  int active_child[TCG_MAX_NODES];
  int passive_child[TCG_MAX_NODES];
  int parent[TCG_MAX_NODES];
  int dp_order[TCG_MAX_NODES];
} tcg_plan;

/* templates.hpp:249-259 partition (validated as make_template does, :80-90) */
int tcg_partition(int k, const int32_t* edges, int root, tcg_plan* out);
/* templates.hpp:326-339 automorphism_count */
int tcg_automorphisms(int k, const int32_t* edges, uint64_t* out);
/* color_index.hpp:103-180 build_split_table: by-parent (active_index,
 * passive_index [C(k,ps) * C(ps,as)]) and grouped (grouped_parent,
 * grouped_active [C(k,ps-as) * C(k-(ps-as),as)]) views; any may be NULL. */
int tcg_split_table(int k, int parent_size, int active_size, int32_t* active_index,
                    int32_t* passive_index, int32_t* grouped_parent, int32_t* grouped_active);
/* color_index.hpp:44-56 / 60-72 */
int64_t tcg_color_index_of(int k, const int32_t* colors, int h);
int tcg_color_set_of(int k, int64_t index, int h, int32_t* colors);
/* count_table.hpp:113-133 estimate_bytes (the reference's fp64 model) */
int64_t tcg_estimate_bytes(const tcg_plan* plan, int64_t n);
/* estimator.hpp:29-33 */
double tcg_colorful_probability(int k);
/* Rooted-color compression layout of a size-s sub-template table (B200
 * design, no reference counterpart): info[4] = {zw, groups,
 * full_cols, store_cols}; optional perm[full_cols] (full column -> P' storage
 * column) and slot_col[k * groups * zw] (compressed slot -> full column or -1). */
int tcg_rooted_layout(int k, int s, int32_t* info, int32_t* perm, int32_t* slot_col);
/* Host-only self-check of the work layout of the vertex-per-CTA blocked eMA (k = 15/17 nodes; B200
 * design, no reference counterpart): the (k, s, a) problem over V vertices per pass is
 * cut into tasks of 32 / V same-shape output groups; every (group, block) of the split enumeration
 * must appear exactly once at the position the kernel reads (TCG_ELOGIC otherwise).  info[6] =
 * {tasks, groups, block steps, pattern runs, shared-load wavefronts of the chosen block order,
 * conflict-free wavefronts}. */
int tcg_rtv_task_layout(int k, int s, int a, int V, int64_t* info);

/* ------------------------------------------------------------------------
 * Device engine (one GPU).  == the vectorized engine of engines.hpp:224-268.
 * ---------------------------------------------------------------------- */
typedef struct tcg_ctx tcg_ctx;

typedef struct {
  int device;              /* CUDA ordinal */
  int64_t memory_budget;   /* bytes of device tables; 0 = unlimited
                              (EngineConfig::memory_budget, engines.hpp:48) */
  int flags;               /* TCG_KEEP_TABLES: keep every node table and SpMM
                              output of the last coloring for inspection */
  int reserved[5];
} tcg_config;

#define TCG_KEEP_TABLES 1

/* NodeStats (engines.hpp:53-61) + device time. */
typedef struct {
  double seconds;            /* CUDA-event time of the node's kernels */
  double spmm_seconds;
  double ema_seconds;
  uint64_t neighbor_passes;  /* one per passive column (pruned/vectorized) */
  uint64_t traversals;       /* neighbor_passes * n */
  uint64_t flops;            /* reference counting: C_p*nnz + 2*n*pairs */
  uint64_t spmm_bytes;       /* SURVEY 8(d) algorithmic bytes */
  uint64_t ema_bytes;
  uint64_t ema_flops;
} tcg_node_stats;

int tcg_create(const tcg_config* cfg, tcg_ctx** out);
/* One context over several GPUs of this process (the reference's
 * run_iteration/estimate use the whole machine through their WorkerPool,
 * engines.hpp:302-307): every device holds the graph and the template, and
 * tcg_estimate / tcg_time_colorings spread the colorings seed+i over the
 * devices in contiguous chunks (one host thread per device, no collective;
 * totals in i order, the reference's estimator arithmetic).  Single-coloring
 * and inspection calls run on device_ids[0].  Graphs too large for one GPU
 * are vertex-sharded instead: one context per rank + tcg_set_shard_nccl. */
int tcg_create_multi(const tcg_config* cfg, const int* device_ids, int ndev, tcg_ctx** out);
int tcg_device_count_of(const tcg_ctx* ctx);
void tcg_destroy(tcg_ctx* ctx);

/* Upload the graph (copied host -> device; builds the SpMM row schedule). */
int tcg_set_graph(tcg_ctx* ctx, int32_t n, const int64_t* row_ptr, const int32_t* col);
int tcg_set_graph_handle(tcg_ctx* ctx, const tcg_graph* g);
/* graph.hpp:65-95 from_edges ON THE DEVICE: m raw (u,v) int32 pairs (any
 * direction, duplicates and self-loops allowed) -> the reference's CSR
 * (symmetric union, no loops, no duplicates, rows ascending) built by a
 * radix sort + dedup on the GPU; n_hint < 0 = max id + 1.  Ids out of range
 * -> TCG_EPARSE ("vertex id out of range [0, n)"), as the reference. */
int tcg_set_graph_edges(tcg_ctx* ctx, const int32_t* edges, int64_t m, int32_t n_hint);
/* The context's graph as a CSR over the caller's vertex ids (inspection):
 * *n, *nnz, row_ptr[n+1] and col[nnz] -- every pointer nullable. */
int tcg_get_graph_csr(tcg_ctx* ctx, int32_t* n, int64_t* nnz, int64_t* row_ptr, int32_t* col);
/* Validate + partition + split tables + |Aut| on the host; upload tables. */
int tcg_set_template(tcg_ctx* ctx, int k, const int32_t* edges, int root);
/* Device bytes one coloring needs (arena peak + graph + schedules). */
int tcg_required_device_bytes(tcg_ctx* ctx, int64_t* bytes);
int tcg_get_plan(tcg_ctx* ctx, tcg_plan* out, uint64_t* aut);

/* count_table.hpp:90-99 random_coloring, generated ON DEVICE
 * (MT19937-64 + rejection), bit-exact; colors = n bytes. */
int tcg_coloring(tcg_ctx* ctx, uint64_t seed, uint8_t* colors);

/* One coloring == run_iteration(vectorized, ..., keep_full_table).
 * colors != NULL: use the caller's coloring (Coloring argument of
 * run_iteration); else generate on device from `seed`.
 * per_vertex (n doubles, nullable) = M_root[:,0]; stats (num_nodes entries
 * indexed by plan node id, nullable). */
int tcg_run_coloring(tcg_ctx* ctx, uint64_t seed, const uint8_t* colors, double* rooted_total,
                     double* per_vertex, tcg_node_stats* stats);

/* == estimate(): colorings seed, seed+1, ... (estimator.hpp:66).
 * rooted_totals[iterations]; per_vertex_estimate (n, nullable) =
 * mean_i M_root^(i)[v,0] / (aut * k!/k^k). */
int tcg_estimate(tcg_ctx* ctx, uint64_t seed, int iterations, double* rooted_totals,
                 double* estimate, double* stderr_of_mean, double* per_vertex_estimate);

/* Inspection (TCG_KEEP_TABLES): node table of the last coloring as
 * vertex-major fp64 n x C(k,|T_s|); which = 0 node table, 1 the SpMM output
 * P' computed from it (passive children only).  Root: C = 1.  P'[v, T] is
 * only computed where T misses c(v) -- the only columns any eMA reads, since
 * M_a[v, Sa] = 0 unless c(v) is in Sa -- and exported as 0 elsewhere. */
int tcg_node_table(tcg_ctx* ctx, int node_id, int which, double* out);
/* Kernel-level hook: Y = A X for a vertex-major fp32 n x C host matrix,
 * through the production SpMM kernel (la_kernels.hpp:83-102 semantics). */
int tcg_spmm(tcg_ctx* ctx, const float* x, int cols, float* y);
/* Kernel-level hook of the PRODUCTION rooted SpMM of one DP node (the
 * la_kernels.hpp:83-102 SpMM as every coloring runs it): x = a passive table
 * M, vertex-major fp32 n x C(k,s), rooted (M[u,S] = 0 unless colors[u] is in
 * S); it goes through the per-coloring colour bucketing, the k-colour slot
 * layout (pair = 0) or the pair layout (pair = 1: per-row-colour copies), the
 * spmm_rooted kernel and the split-row fixup.  y (n x C(k,s)) receives
 * Y[v,T] = sum over u in N(v) of M[u,T] wherever T misses colors[v] -- the
 * columns a consumer reads -- and 0 elsewhere.  2 <= k <= 20, 1 <= s < k. */
int tcg_spmm_rooted(tcg_ctx* ctx, int k, int s, int pair, const uint8_t* colors, const float* x, float* y);
/* Test hook: override the rejection threshold (UINT64_MAX/k)*k of
 * Rng::below (rng.hpp:21-27); 0 restores the reference value. */
int tcg_set_rejection_limit(tcg_ctx* ctx, uint64_t limit);
/* Device-timed batch of colorings (bench.py's timed region): colorings
 * seed..seed+count-1 generated on device and run back to back on the
 * engine's stream, bracketed by CUDA events recorded ON THAT STREAM.  With
 * per_kernel != 0 every SpMM / eMA launch is additionally bracketed so the
 * phase times below are measured (otherwise they are 0).  Rooted totals
 * land in totals[count] (nullable). */
typedef struct {
  double total_ms;            /* device time of the whole batch */
  double spmm_ms, ema_ms;     /* summed over launches (per_kernel) */
  int64_t spmm_launches, ema_launches, launches;
  double spmm_alg_bytes;      /* 4 nnz + 8 (n+1) + 8 n C_p per internal passive */
  double hist_alg_bytes;      /* leaf passives: 4 nnz + 8 (n+1) + n + 4 n k, once per coloring */
  double ema_alg_bytes;       /* 4 n (C_a + C_p + C_s), root writes 8 n */
  double ema_flops;           /* 2 n C_s C(|T_s|,|T_a|) */
  double spmm_gathered_bytes; /* bytes moved L2 -> SM by the panel gathers: nnz * 64 B * panels */
} tcg_timing;
int tcg_time_colorings(tcg_ctx* ctx, uint64_t seed, int count, int per_kernel, double* totals,
                       tcg_timing* out);

/* ------------------------------------------------------------------------
 * Vertex sharding: the context owns a contiguous range of
 * vertex rows (balanced by degree + average degree); every count table holds
 * only those rows (padded to the largest shard), and before each SpMM panel
 * the passive table's panel is all-gathered from every rank.  eMA is local;
 * rooted totals are summed in rank order on the host (deterministic).
 * Call before tcg_set_graph.  All ranks call the same entry points with the
 * same arguments (graph, template, seeds).
 * ---------------------------------------------------------------------- */
/* Row bounds of each shard: bounds[world+1] (host-only, no GPU needed). */
int tcg_shard_bounds(int32_t n, const int64_t* row_ptr, int world, int64_t* bounds);
/* All-gather callback: `send` holds this rank's `bytes`, `recv` receives
 * world*bytes in rank order.  Returns 0 on success. */
typedef int (*tcg_allgather_fn)(void* user, const void* send, size_t bytes, void* recv);
/* Device transport (production): send/recv are DEVICE pointers, the engine
 * stream is synchronized before the call and recv must be complete on return
 * (e.g. torch.distributed.all_gather_into_tensor, NCCL over NVLink/NVSwitch). */
int tcg_set_shard_device(tcg_ctx* ctx, int rank, int world, tcg_allgather_fn fn, void* user);
/* Host transport (tests, any backend): send/recv are HOST buffers. */
int tcg_set_shard_host(tcg_ctx* ctx, int rank, int world, tcg_allgather_fn fn, void* user);
/* NCCL data plane owned by the library (production, one process per GPU):
 * rank 0 calls tcg_nccl_unique_id, the caller hands the 128 bytes to every
 * rank (any side channel: torch.distributed, MPI, a file), and each rank
 * calls tcg_set_shard_nccl.  The library creates its own communicator
 * (ncclCommInitRank over the process's NCCL, resolved at run time) and
 * enqueues every panel all-gather on a communication stream, double-buffered
 * against the SpMM of the previous group -- no host synchronization per panel. */
#define TCG_NCCL_ID_BYTES 128
/* In-process loopback transport: `world` contexts of THIS process (several may
 * share one GPU) act as the ranks; panels move by device-to-device copies
 * enqueued asynchronously exactly like the NCCL transport's all-gathers (so
 * the pipelined sharded SpMM runs with world > 1 on one GPU).  Every rank's
 * calls must come from its own host thread, concurrently (the hub's host
 * barriers order the ranks' enqueues; no kernel waits on another rank). */
typedef struct tcg_loopback tcg_loopback;
int tcg_loopback_create(int world, tcg_loopback** out);
void tcg_loopback_destroy(tcg_loopback* hub);   /* after every context using it */
int tcg_set_shard_loopback(tcg_ctx* ctx, int rank, tcg_loopback* hub);
int tcg_nccl_unique_id(uint8_t id[TCG_NCCL_ID_BYTES]);
int tcg_set_shard_nccl(tcg_ctx* ctx, int rank, int world, const uint8_t id[TCG_NCCL_ID_BYTES]);

/* Kernel launches issued by this context since creation (evidence for
 * bench.py's gpu_launches). */
int64_t tcg_kernel_launches(const tcg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TCG_H */

/*
 * tc_oracle.h -- CPU restatement of the reference's pruned color-coding DP.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 path;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
 * legs may load it.  The product (paper_1903_04395_b200/) never links it.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/proj/include/treecount/) in plain C99 with fp64 tables,
 * in the reference's own arithmetic order, so per-node tables and rooted
 * totals are bit-identical to EngineKind::vectorized built with the
 * reference's flags (-O3, no -march; SURVEY finding 10).  Pinned against the
 * compiled reference (oracle/_ref) and the golden vectors in tests/golden/.
 */
#ifndef TC_ORACLE_H
#define TC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- rng.hpp:13-37: std::mt19937_64 + rejection below() ----------------- */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;
void     orc_mt_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt_next(orc_mt64* g);
/* count_table.hpp:90-99.  limit_override != 0 replaces (UINT64_MAX/k)*k
 * (test hook that forces the rejection path; 0 = reference behaviour). */
void     orc_random_coloring(int32_t n, int k, uint64_t seed, uint64_t limit_override,
                             uint8_t* out);

/* --- graph.hpp:46-95: symmetrize, drop self-loops, dedup, sort, CSR ------ */
/* edges: m (u,v) int32 pairs.  n_hint<0 -> max id + 1.  Returns 0 or -1 (id
 * out of range).  *row_ptr (n+1) and *col (nnz) are malloc'd; free with
 * orc_free. */
int  orc_csr_from_edges(const int32_t* edges, int64_t m, int32_t n_hint, int32_t* n_out,
                        int64_t** row_ptr, int32_t** col, int64_t* nnz);
/* synthgen.hpp:40-74 (R-MAT, harness input generator) */
int  orc_generate_rmat(int scale, int64_t nedges, double a, double b, double c, double d,
                       uint64_t seed, int32_t* n_out, int64_t** row_ptr, int32_t** col,
                       int64_t* nnz);
void orc_free(void* p);

/* --- color_index.hpp:20-82 ---------------------------------------------- */
int64_t orc_binom(int a, int b);
int64_t orc_index_of(const int* colors, int h);
void    orc_set_of(int k, int64_t index, int h, int* colors);

/* --- color_index.hpp:103-180: split table for one internal node --------- */
/* by-parent view [I_s*pairs + p] and grouped view [I_p*partners + q]. */
int orc_split_table(int k, int parent_size, int active_size, int32_t* active_index,
                    int32_t* passive_index, int32_t* grouped_parent, int32_t* grouped_active);

/* --- templates.hpp:37-90,174-259: validation, default root, partition ---- */
#define ORC_MAXK 20
#define ORC_MAXNODES (2 * ORC_MAXK - 1)
typedef struct {
  int k, root, num_nodes;
  int size[ORC_MAXNODES];
  int node_root[ORC_MAXNODES];
  int active_child[ORC_MAXNODES], passive_child[ORC_MAXNODES], parent[ORC_MAXNODES];
  int dp_order[ORC_MAXNODES];
} orc_plan;
/* edges: k-1 pairs; root<0 -> default_root.  Returns 0, or -1 (not a tree). */
int orc_partition(int k, const int32_t* edges, int root, orc_plan* plan);
/* templates.hpp:326-339 (AHU at the tree centers) */
uint64_t orc_automorphisms(int k, const int32_t* edges);
/* count_table.hpp:113-133 */
int64_t orc_estimate_bytes(const orc_plan* plan, int64_t n);

/* --- engines.hpp:106-132,224-268 + la_kernels.hpp:50-114 ----------------- */
/* One coloring through the vectorized engine, fp64.  per_vertex (n, nullable)
 * receives M_root[:,0]; node_tables (nullable, indexed by plan node id) gets
 * a malloc'd column-major n x C(k,|T_s|) copy of every node's table as it is
 * when its parent consumes it (internal nodes) -- passive children are
 * captured BEFORE their in-place SpMM.  Returns the rooted total. */
double orc_run_iteration(int32_t n, const int64_t* row_ptr, const int32_t* col,
                         const orc_plan* plan, const uint8_t* colors, double* per_vertex,
                         double** node_tables);

/* --- estimator.hpp:29-33,49-93 ------------------------------------------ */
double orc_colorful_probability(int k);
void   orc_estimate(int32_t n, const int64_t* row_ptr, const int32_t* col, int k,
                    const int32_t* edges, int root, int iterations, uint64_t seed,
                    double* rooted_totals, double* estimate, double* stderr_of_mean,
                    uint64_t* aut);

#ifdef __cplusplus
}
#endif
#endif

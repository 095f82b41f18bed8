/* ============================================================================
 * pilotann.h — C ABI of the B200-native PilotANN GPU stage (arXiv 2503.21206).
 *
 * The boundary follows the paper's statement of the problem: top-k search of a
 * query q over a graph with entry points and candidate size ef (PAPER.md
 * P:L181-182, Alg 1), with PilotANN's GPU stage in front of it (§4.1 ①, §5):
 *
 *   build(subgraph, reduced vectors, SVD basis [, FES entry index])   pa_build
 *   search(queries, k, ef) -> top-k ids and distances                  pa_search
 *
 * Citations: P:Lnnn = PAPER.md line; S:Lnnn = SPEC.md line; SURVEY §8.b/§8.c.
 *
 * Conventions for every call
 *   - Every call returns pa_status; no C++ exception crosses the ABI.  On
 *     failure pa_last_error() returns a thread-local message, valid until the
 *     next call on that thread.
 *   - "host" pointers are ordinary CPU memory (pageable or pinned);
 *     "device" pointers are CUDA global memory on the index's device.
 *   - Ids are int32 in the FULL graph id space (modified CSR):
 *     non-members keep their id, have empty adjacency rows and are never
 *     returned.  Vectors are row-major fp32.
 *   - Distances: PA_L2 = squared Euclidean, no sqrt;
 *     PA_IP = negative inner product (−q·x), so smaller is better for both.
 *     Results are ordered by (distance, id) ascending (Q13); rows with fewer
 *     than k valid results are padded with id −1 and distance +inf (Q26).
 *   - One search at a time per index: calls serialise on an internal mutex,
 *     and on the device every search (whatever stream it is enqueued on) waits
 *     for the end of the previous one, because they share the index's device
 *     workspace; separate indexes are independent.  One process per GPU is the
 *     intended multi-GPU layout: each process builds its own replica with
 *     params.device and searches its shard of the queries.
 * ========================================================================== */
#ifndef PILOTANN_H_
#define PILOTANN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PA_OK = 0,
    PA_EINVAL = -1,  /* null pointer / bad size / k<1 / ef<k / rdim>dim / max_degree>64 / ef1>256 / ef2,ef3>512 / non-finite */
    PA_EGRAPH = -2,  /* CSR invalid: offsets[0]!=0, non-monotone, id out of range, self-loop, duplicate,
                        degree>max_degree, edge into a non-member, non-member with edges */
    PA_EBASIS = -3,  /* basis not orthonormal: max|VᵀV − I| > 1e-4 */
    PA_EFES = -4,    /* FES index invalid: empty cell, pool id not a member / out of range / duplicated */
    PA_ENOMEM = -5,  /* device or pinned allocation failed */
    PA_ECUDA = -6,   /* other CUDA error (message carries cudaGetErrorString) */
    PA_ESTATE = -7,  /* bad handle (destroyed / not built) or stage ②③ requested without pa_attach_host */
    PA_ENOTSUP = -8, /* unsupported option, or a query exceeded the exact visited-set capacity */
} pa_status;

typedef enum { PA_L2 = 0, PA_IP = 1 } pa_metric;

typedef enum {
    PA_STAGES_GPU = 1,  /* stage ① only: FES + subgraph traversal on reduced vectors (§4.1 ①, §5)  */
    PA_STAGES_FULL = 3, /* ① on the GPU, then ② residual refinement and ③ final traversal on host   */
    PA_STAGES_FULL_GPU = 7, /* NEXT-f3: ①②③ all on the GPU (O8-O9 semantics, exact visited sets in ②③);
                               needs pa_attach_host, whose full graph (degree ≤ 64) and X̂ are copied to
                               the device on first use (PA_ENOMEM if they do not fit) */
} pa_stages;

/* Ablation toggles (Table 6). */
enum {
    PA_NO_FES = 1u,    /* entries = the first E pool ids in pool order (no routing / scoring)   */
    PA_NO_STAGE2 = 2u, /* carry = stage-① candidates re-ranked by full δ, visited = their ids      */
    PA_NO_STAGE1 = 4u, /* stage-① output = the entries themselves (no subgraph traversal)        */
    PA_NO_PIPELINE = 8u, /* PA_STAGES_FULL: run the GPU stage over the whole batch before the host
                            stages start (no CPU–GPU overlap, Table 6 "−pipelining"); results identical */
};

typedef struct pa_index pa_index; /* opaque */

/* Inputs of pa_build.  All pointers are HOST pointers; pa_build copies what it
 * needs (device replica + a host copy of the subgraph CSR for stage ②), so the
 * caller may free them on return. */
typedef struct {
    int64_t n;                     /* nodes in the full id space (< 2^31)                        */
    int32_t dim;                   /* D, full dimension                                          */
    int32_t rdim;                  /* d', reduced dimension, 1 ≤ d' ≤ D                 */
    int32_t max_degree;            /* bound on subgraph out-degree, 1..64 (R = 32 default) */
    int32_t metric;                /* pa_metric                                                  */
    const int64_t* sub_offsets;    /* [n+1] sampled subgraph CSR over the full id space            */
    const int32_t* sub_neighbors;  /* [sub_offsets[n]] neighbour ids; row order = visit order      */
    const uint8_t* member_flags;   /* [n] 1 = sampled member; NULL ⇒ member iff degree>0 */
    const float* reduced;          /* [n][rdim] x_primary = rows of X·V[:, :rdim]; non-member rows ignored */
    const float* basis;            /* [dim][dim] orthonormal V, columns by descending singular value */
    int32_t fes_r;                 /* r FES cells, 1..1024 (r = 32 in the paper)         */
    const float* fes_centroids;    /* [fes_r][rdim]                                              */
    const int64_t* fes_cell_off;   /* [fes_r+1] pool offsets per cell; every cell non-empty       */
    const int32_t* fes_pool_ids;   /* [fes_cell_off[fes_r]] member ids grouped by cell */
    int32_t device;                /* CUDA device ordinal of this replica                         */
    int32_t reduced_fp16;          /* NEXT-f1: 1 = store the reduced rows as IEEE binary16,
                                      rounded once (RNE) at build; stage ① and the FES pool then use
                                      exactly these rounded values (half the gather bytes); stage ②
                                      recomputes full δ from X̂.  0 = fp32 rows (default)            */
    int64_t reduced_stride;        /* floats between consecutive rows of `reduced` (0 ⇒ rdim).  With
                                      stride = dim the caller passes X̂ itself: x_primary is exactly the
                                      first d' columns of X̂ = X·V, so a 100M-row index
                                      needs no separate [n][d'] host copy.  Must be ≥ rdim (PA_EINVAL). */
} pa_build_params;

/* Per-call options; pass NULL for defaults.  Zero fields take defaults
 * (SURVEY §8.0, Q21): ef1 = ef3 = ef, ef2 = max(k, ef/2), entries E = ef1,
 * width w = 1 (Alg 1), refine_iters = 2. */
typedef struct {
    int32_t stages;          /* pa_stages (0 ⇒ PA_STAGES_GPU)                                 */
    int32_t ef1, ef2, ef3;   /* per-stage candidate capacities: ef1 ≤ 256 (stage ①'s lists),
                                ef2, ef3 ≤ 512 (stages ②③; pass ef1 explicitly when ef > 256)    */
    int32_t entries;         /* E entries seeded into C per query (Q8)                          */
    int32_t width;           /* search width w, 1..8 (SURVEY §8.c O6 generalisation of Alg 1: the w
                                smallest unchecked entries are expanded per iteration, rows visited in
                                key order; all three stages).  w > 1 runs the sequential kernel with
                                the exact visited set (PA_ENOTSUP with bloom_log2 > 0)            */
    int32_t refine_iters;    /* stage-② expansions (−1 ⇒ 0 iterations; 0 ⇒ default 2)          */
    uint32_t flags;          /* PA_NO_* ablation toggles                                       */
    int32_t hash_slots_log2; /* visited-hash smem slots = 2^this (0 ⇒ auto); test hook for spill */
    int32_t host_threads;    /* threads for stages ②③ (0 ⇒ env PILOTANN_HOST_THREADS or all cores) */
    int32_t bloom_log2;      /* NEXT-f1, the paper's own visited set: 0 ⇒ EXACT visited set;
                                s in 7..16 ⇒ stage ① tracks visited nodes in a shared-memory bloom filter of
                                3 segments × 2^s bits (segment j: bit ((uint32)v·A_j) >> (32−s), A = 0x9E3779B1,
                                0x85EBCA77, 0xC2B2AE3D).  False positives skip nodes (stages ②③ keep exact
                                sets and re-visit); results then match the oracle's O13 mode.
                                Requires max_degree ≤ 32 (PA_ENOTSUP otherwise); other values PA_EINVAL. */
    uint32_t check_path;     /* test hooks that select a cross-check implementation (results must not change):
                                PA_CHECK_SIMT = run the SIMT fp32 projection + FES kernels instead of the tcgen05
                                ones; PA_CHECK_WIDE_VISITED = 32-bit exact visited table even when ids < 2^24.
                                0 for normal use. */
} pa_search_opts;

enum { PA_CHECK_SIMT = 1u, PA_CHECK_WIDE_VISITED = 2u };

/* Optional per-query debug/trace outputs of stage ① (DEVICE pointers, may be
 * NULL individually).  Trace mode is for parity tests, never for timed runs. */
typedef struct {
    int32_t* cell;          /* [m]         routed FES cell                          */
    int32_t* entries;       /* [m][E]      FES-selected entry ids, −1 padded                  */
    int32_t* cand_ids;      /* [m][ef1]    final stage-① candidate list C (ids)               */
    float* cand_dists;      /* [m][ef1]    reduced-space δ' of C                              */
    int32_t* counters;      /* [m][4]      n_exp, n_dist, spill_inserts, status (0 ok, 1 overflow, 2 iter cap) */
    int32_t trace_cap;      /* per-query capacity of the two traces below                       */
    int32_t* trace_expand;  /* [m][trace_cap] expansion sequence (Alg 1 l.5)                   */
    int32_t* trace_visit;   /* [m][trace_cap] visit sequence (Alg 1 l.7), entries first          */
    int32_t* trace_nexp;    /* [m] full lengths (may exceed trace_cap)                          */
    int32_t* trace_nvis;    /* [m]                                                              */
} pa_debug;

/* Timings and counters of the last search on this index. */
typedef struct {
    int64_t queries;
    int64_t kernel_launches;     /* product kernels launched by the last search            */
    double ms_project, ms_fes, ms_traverse, ms_total_gpu; /* device time (CUDA events)      */
    double ms_h2d, ms_d2h, ms_host_stages, ms_wall;      /* host-observed                  */
    int64_t sum_n_exp, sum_n_dist, sum_spill;            /* stage ① counters, summed        */
    int64_t overflow_queries;                            /* queries that hit a cap           */
    int64_t sum_n_dist2, sum_n_dist3;                    /* stages ②③ (host, or GPU)       */
    double ms_refine;                                    /* PA_STAGES_FULL_GPU: ②③ kernel  */
} pa_stats;

/* Build one device replica.  Validates every input (PA_EINVAL / PA_EGRAPH /
 * PA_EBASIS / PA_EFES) BEFORE touching the GPU, converts the subgraph to a
 * −1-padded ELL [n][32 or 64], groups FES pool vectors by cell, and uploads.
 * On success *out owns all device memory, streams and events. */
pa_status pa_build(const pa_build_params* p, pa_index** out);

/* Borrow the host-resident full graph (CSR over the same n ids, any degree)
 * and the rotated full vectors X̂ = X·V [n][dim] for stages ②③.
 * They must stay alive and unchanged until pa_destroy.  Validates the CSR. */
pa_status pa_attach_host(pa_index* ix, const int64_t* full_offsets, const int32_t* full_neighbors,
                         const float* rotated_full);

/* End-to-end search of m HOST query rows [m][dim]: H2D (pinned staging) →
 * projection → FES → traversal → D2H, then (PA_STAGES_FULL) host stages ②③.
 * Writes out_ids/out_dists [m][k] (HOST).  PA_STAGES_GPU returns reduced-space
 * δ' (top-k of stage ①'s C); PA_STAGES_FULL returns full-space δ over X̂ and
 * requires pa_attach_host (else PA_ESTATE).  Errors: PA_EINVAL for k<1, ef<k,
 * ef1>256 or ef2/ef3>512 (after defaults), m<0, null pointers. */
pa_status pa_search(pa_index* ix, const float* queries, int64_t m, int32_t k, int32_t ef,
                    const pa_search_opts* opts, int32_t* out_ids, float* out_dists);

/* GPU stage only, all arrays DEVICE-resident on the index's device, enqueued on
 * `stream` (a cudaStream_t; NULL = the legacy default stream) and NOT
 * synchronised: q [m][dim] → out_ids/out_dists [m][k] (reduced δ'), plus the
 * optional debug outputs.  This is the call bench.py times with inputs already
 * resident in HBM. */
pa_status pa_search_device(pa_index* ix, const float* d_queries, int64_t m, int32_t k, int32_t ef,
                           const pa_search_opts* opts, int32_t* d_out_ids, float* d_out_dists,
                           const pa_debug* dbg, void* stream);

/* Stage-① candidate lists for HOST queries: cand_ids/cand_dists [m][ef] (HOST),
 * i.e. what the GPU hands to the host stages ("<1KB per query").
 * opts->stages must be 0 or PA_STAGES_GPU (PA_EINVAL otherwise). */
pa_status pa_search_candidates(pa_index* ix, const float* queries, int64_t m, int32_t ef,
                               const pa_search_opts* opts, int32_t* cand_ids, float* cand_dists);

/* Entry selection alone (NEXT-f4, the "FES analysis" of §6.3): the
 * E entry ids of m DEVICE query rows [m][dim], enqueued on `stream`, not
 * synchronised, written to d_entries [m][E] (DEVICE, −1 padded).
 *   PA_ENTRIES_FES     : projection + FES exactly as pa_search's stage ① seeds
 *                        (a1–a4); entries in ascending (score, id).
 *   PA_ENTRIES_TWO_HOP : projection + the two-hop baseline (oracle O14): from
 *                        node e0, hop 1 visits N(e0), hop 2 the neighbours of the
 *                        `beam` nearest hop-1 nodes; entries = the E smallest
 *                        (δ', id) over every visited node, ascending.  d_entry_dists
 *                        [m][E] (δ', +inf padded) and d_n_dist [m] (nodes visited)
 *                        are optional (NULL).
 * Errors: PA_EINVAL for E < 1, E > 256, beam < 0, e0 outside [0, n), null
 * pointers, an unknown method; PA_ENOTSUP for TWO_HOP on a max_degree-64 or
 * binary16 index.  pa_get_stats reports ms_project and ms_fes (= the selection). */
typedef enum { PA_ENTRIES_FES = 0, PA_ENTRIES_TWO_HOP = 1 } pa_entry_method;
pa_status pa_entries_device(pa_index* ix, const float* d_queries, int64_t m, int32_t E, int32_t method,
                            int32_t e0, int32_t beam, int32_t* d_entries, float* d_entry_dists,
                            int32_t* d_n_dist, void* stream);

/* ---------------------------------------------------------------------------
 * Replication across GPUs: queries are independent, so
 * every GPU holds a full replica of the device index and searches its own shard.
 * The index is built ONCE (pa_build on the first GPU); the other processes
 * allocate an empty replica with the same layout and receive the device arrays
 * over NVLink (e.g. an NCCL broadcast of every buffer pa_replica_buffers lists).
 * A replica has no host copy of the subgraph, so it serves PA_STAGES_GPU and
 * PA_STAGES_FULL_GPU (if the source had uploaded the full graph and X̂ before
 * its meta was exported) but not the host stages (PA_ESTATE).
 * ------------------------------------------------------------------------- */
typedef struct {
    int64_t n, pool_n;
    int32_t dim, rdim, rdim_pad, rdim_h, qlen, rstride, rstride_h, ell_w, metric, fes_r;
    int32_t max_cell, proj_nb, pool_chunks, fes_fold_norm, reduced_fp16;
    int32_t has_full, full_w, xstride;    /* device copies of the full graph and X̂ (NEXT-f3) */
} pa_replica_meta;

typedef struct {
    void* ptr;       /* DEVICE pointer on the index's device */
    int64_t bytes;
} pa_buffer;

/* Layout of a built index (PA_ESTATE on a bad handle). */
pa_status pa_replica_meta_of(const pa_index* ix, pa_replica_meta* out);

/* Allocate an EMPTY replica with the layout `meta` on `device` (contents
 * undefined until every buffer of pa_replica_buffers has been filled with the
 * source's bytes).  PA_EINVAL for an inconsistent meta, PA_ENOMEM if it does not fit. */
pa_status pa_build_replica(const pa_replica_meta* meta, int32_t device, pa_index** out);

/* The index's read-only device arrays, in a fixed order that is identical for
 * a source and a replica of the same meta: writes min(cap, total) entries of
 * out[] and the total count to *count. */
pa_status pa_replica_buffers(pa_index* ix, pa_buffer* out, int32_t cap, int32_t* count);

/* Copy the last search's pa_stats into *out (size = sizeof(pa_stats)). */
pa_status pa_get_stats(const pa_index* ix, pa_stats* out, size_t size);

/* Release everything.  NULL-safe; a second destroy of the same handle is
 * detected by a magic field and ignored. */
void pa_destroy(pa_index* ix);

const char* pa_last_error(void);
const char* pa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PILOTANN_H_ */

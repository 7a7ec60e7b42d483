/*
 * hifuse.h -- C ABI of the B200 (sm_100a) HiFuse hot path.
 *
 * HiFuse (arXiv 2408.08490) speeds up mini-batch HGNN training by merging the
 * per-semantic-graph work of every HGNN layer.  A layer has four stages
 * (PAPER.md lines 112-125): semantic graph build, feature projection,
 * neighbour aggregation, semantic fusion.  This library runs all four on the
 * GPU, each as a small, fixed number of kernels that does not grow with the
 * number of relations R:
 *
 *   hifuse_build_semantic_graphs  Alg. 2 (lines 310-324) + merging: one
 *                                 segmented CSR over all relations (and its
 *                                 CSC transpose); integer work, bit-exact.
 *   hifuse_project                per-relation / per-type projection (line 119),
 *                                 one grouped GEMM launch; layer 0 gathers its
 *                                 rows from the type-major feature store
 *                                 (reorganisation, lines 199-221).
 *   hifuse_aggregate_fwd          Alg. 1 (lines 246-262): ONE gather-reduce
 *                                 kernel for every relation (sum / mean / GAT
 *                                 edge softmax).
 *   hifuse_semantic_fuse          fusion (line 123): sum over relations + root
 *                                 + bias, activation.
 *   *_bwd                         the adjoints (line 156, "backward pass on GPU
 *                                 for gradient computation").
 *
 * Conventions:
 *  - Pointers named d_* are device memory; *_h are host memory.  The caller
 *    owns every buffer, including workspace; the library never allocates
 *    device memory.  Its only state: cached device attributes (SM count,
 *    per-kernel shared-memory opt-in) and, per (device, caller stream), the
 *    auxiliary streams + events that fork a call's independent kernels into
 *    parallel branches (see hifuse_stream_attach).  Calls on different
 *    streams share none of it; calls on one stream must come from one host
 *    thread at a time (as stream order already requires).
 *  - Every call is asynchronous and stream-ordered on `stream`; no call
 *    synchronises the device (except hifuse_read_status, for tests).  All
 *    sizes a launch needs are host-known from hifuse_layer_shape, so a whole
 *    step is CUDA-graph capturable; the one data-dependent size, the number U
 *    of rows of the merged projected matrix, lives in device memory (U_dev).
 *  - fp32 row-major everywhere; feature widths K, D must be 64 or 128
 *    (HIFUSE_ERR_UNSUPPORTED otherwise); heads H must divide D with D/H a
 *    multiple of 4.  int32 local ids and offsets (N < 2^31), int64 edge ids.
 *  - Host-detectable errors (null pointer, bad sizes, misalignment) return
 *    synchronously and launch nothing.  Data errors found on the device
 *    (edge id out of range, relation id out of range, local id out of range)
 *    OR bits into *d_status (HIFUSE_ST_*) and the offending edge is dropped:
 *    no out-of-bounds access ever happens.
 *  - Results are deterministic: the build is bit-exact against the CPU oracle
 *    (oracle/hifuse_oracle.c), reductions use fixed orders, no float atomics.
 */
#ifndef HIFUSE_H
#define HIFUSE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *hifuse_stream_t;   /* == cudaStream_t */

typedef enum {
  HIFUSE_OK = 0,
  HIFUSE_ERR_INVALID_ARG = 1,   /* null pointer / negative or inconsistent size */
  HIFUSE_ERR_ALIGNMENT = 2,     /* a float pointer is not 16-byte aligned       */
  HIFUSE_ERR_UNSUPPORTED = 3,   /* K, D, H or layout outside the supported set   */
  HIFUSE_ERR_WORKSPACE = 4,     /* ws_bytes smaller than the *_sizes() answer    */
  HIFUSE_ERR_CUDA = 5           /* a CUDA launch failed (cudaGetLastError)       */
} hifuse_status;

/* device status bits (ORed into d_status by the build) */
#define HIFUSE_ST_BAD_EDGE_ID 1   /* edge_id < 0 or >= num_graph_edges          */
#define HIFUSE_ST_BAD_REL     2   /* edge_type[edge_id] not in [0, R)           */
#define HIFUSE_ST_BAD_SRC     4   /* src_local >= n_src(src type of relation)   */
#define HIFUSE_ST_BAD_DST     8   /* dst_local >= n_dst(dst type of relation)   */
#define HIFUSE_ST_UNSORTED_TYPES 16 /* edge_type not relation-major (offsets unusable) */
#define HIFUSE_ST_BAD_LABEL   32  /* class label outside [0, C) (hifuse_linear_xent) */
#define HIFUSE_ST_OVERFLOW    64  /* padded sampler: a block exceeded its capacities  */

/* GAT_XREL: GAT with the edge-softmax across the relations of a destination
 * (hifuse_aggregate_fwd_xrel, reading C5'). */
typedef enum { HIFUSE_AGG_SUM = 0, HIFUSE_AGG_MEAN = 1, HIFUSE_AGG_GAT = 2,
               HIFUSE_AGG_GAT_XREL = 3,
               /* multiplicative attention (reading C23):
                * logit s_src[col] * s_dst[row] per head instead of
                * LeakyReLU(s_src[col] + s_dst[row]); softmax within the row */
               HIFUSE_AGG_GAT_MUL = 4 } hifuse_agg;
typedef enum { HIFUSE_ACT_NONE = 0, HIFUSE_ACT_RELU = 1 } hifuse_act;
/* Layout of the merged projected matrix Y (reading C3).  COMPACT:
 * per relation, one row per distinct source vertex of the layer, ascending.
 * SLOTS (every source vertex x every live relation) is reserved. */
typedef enum { HIFUSE_LAYOUT_SLOTS = 0, HIFUSE_LAYOUT_COMPACT = 1 } hifuse_layout;
/* Projection arithmetic.  FP32: CUDA-core fp32 FMA.  TF32: tcgen05 kind::tf32
 * tensor cores, fp32 accumulate (reading C17/C18).  BF16 (hifuse_project
 * only): X and W rounded to bfloat16 (round-to-nearest-even) on their way
 * into shared memory, tcgen05 kind::f16, fp32 accumulate and fp32 outputs;
 * the RGAT destination scores s_dst stay fp32 (reading C24).  The backward
 * calls take FP32 or TF32. */
typedef enum { HIFUSE_PREC_FP32 = 0, HIFUSE_PREC_TF32 = 1, HIFUSE_PREC_BF16 = 2 } hifuse_prec;

#define HIFUSE_MAX_TYPES 64
#define HIFUSE_MAX_RELS 512

/* Host metadata of one layer's sampled block (Alg. 2 inputs EdgeIndex[i],
 * EdgeID[i] are device arrays passed separately).  Per vertex type t the
 * layer's destination vertices are the first n_dst[t] of its n_src[t] source
 * vertices (reading C12).  Relation r maps type rel_src_type[r] to type
 * rel_dst_type[r].  Derived (host, no sync):
 *   rows = sum_r n_dst[rel_dst_type[r]]   merged (relation, destination) rows,
 *          row (r, i) = rel_row_off[r] + i, relation-major (reading C2);
 *   S    = sum_r n_src[rel_src_type[r]]   (relation, source) slots;
 *   U    <= U_max = min(N, S)             rows of Y (device-resident U_dev). */
typedef struct {
  int32_t num_types, num_rels;
  const int32_t *rel_src_type_h;   /* [R] */
  const int32_t *rel_dst_type_h;   /* [R] */
  const int32_t *n_src_h;          /* [T] */
  const int32_t *n_dst_h;          /* [T] */
  int64_t num_edges;               /* N   */
} hifuse_layer_shape;

/* Caller-allocated device outputs of the build of one layer (int32).
 * CSR: row_ptr over the merged rows; inside a row, edges in ascending original
 * column (Alg. 2 keeps column order); col[p] = Y row read by CSR position p;
 * eperm[p] = original column of position p.  Y rows of relation r are
 * [rel_y_off[r], rel_y_off[r+1]); y_src[u] = source local id of Y row u;
 * slot_y[slot(r, j)] = Y row of (r, j) or -1, slot(r, j) = sum_{r'<r}
 * n_src(src type of r') + j.  CSC over Y rows: col_ptr, csc_pos (CSR
 * position, ascending inside a column), csc_row (merged row of that
 * position), csc_col (the column, i.e. Y row, of the entry: the edge-balanced
 * transpose SpMM reads it instead of searching col_ptr).  Entries past the
 * valid count are -1; col_ptr entries past U equal the number of valid edges.
 * The CSC is optional: col_ptr, csc_pos, csc_row and csc_col all NULL skip
 * the transpose (a layer whose aggregation backward is
 * never run, e.g. the input layer of the aggregate-first RGCN).
 * X-row mode: y_src == NULL (the CSC must then be absent too) skips the Y
 * numbering: col[p] = type_src_off(source type) + source local id, the
 * source's row in the layer's type-major X (what an aggregation over raw
 * rows reads: the aggregate-first input layer); rel_y_off, slot_y and U_dev
 * may be NULL and are not written.  Same rows, positions and eperm. */
typedef struct {
  int32_t *rel_row_off;  /* [R+1]      */
  int32_t *row_ptr;      /* [rows+1]   */
  int32_t *col;          /* [N]        */
  int32_t *eperm;        /* [N]        */
  int32_t *rel_y_off;    /* [R+1]      */
  int32_t *y_src;        /* [U_max]    */
  int32_t *col_ptr;      /* [U_max+1]  */
  int32_t *csc_pos;      /* [N]        */
  int32_t *csc_row;      /* [N]        */
  int32_t *csc_col;      /* [N]        */
  int32_t *slot_y;       /* [S]        */
  int32_t *U_dev;        /* [1]        */
  const int32_t *x_gather; /* X-row mode only, nullable: col[p] = x_gather[X row]
                            * (the feature-store row: the aggregate-first layer
                            * then reads col directly, no hifuse_feature_cols) */
} hifuse_csr;

/* Sizes of one layer (host only, no device work, no sync). */
hifuse_status hifuse_csr_sizes(const hifuse_layer_shape *shape, hifuse_layout layout,
                               int64_t *rows, int64_t *U_max, int64_t *S,
                               size_t *build_ws_bytes);

/* A1. Semantic graph build for `num_layers` layers (Alg. 2 lines
 * 310-324: EdgeTypeLayer = EdgeType[EdgeID], per-relation compare + select),
 * producing the merged segmented CSR/CSC of each layer in `out[l]`.
 *   d_src_local[l], d_dst_local[l]: int32 [N_l] batch-local endpoint ids;
 *   d_edge_id[l]: int64 [N_l] graph-global edge ids; -1 marks a NULL edge
 *     (capacity padding, e.g. the tail of a padded GPU-sampled block): it is
 *     dropped like an invalid edge but sets no status bit;
 *   d_edge_type: int32 [num_graph_edges] relation of every graph edge;
 *   d_rel_edge_off: NULL, or int64 [R+1] with d_edge_type relation-major
 *     (global edge ids sorted by relation): relation r owns ids
 *     [off[r], off[r+1]).  EdgeType[EdgeID] (Alg. 2) is then
 *     evaluated by a binary search over the R+1 offsets instead of a random
 *     4-byte gather from the graph-sized table (same result); build the
 *     offsets once per graph with hifuse_edge_type_offsets().
 * Workspace: d_ws of at least sum_l build_ws_bytes(l) (the layers are built
 * together); no initial contents required.  d_status: int32 [1], bits ORed
 * (never cleared by the library).  Launches: one memset + five kernels for
 * up to 4 layers (build.cu), independent of R and of the layer count. */
hifuse_status hifuse_build_semantic_graphs(const hifuse_layer_shape *shapes, int num_layers,
                                           const int32_t *const *d_src_local,
                                           const int32_t *const *d_dst_local,
                                           const int64_t *const *d_edge_id,
                                           const int32_t *d_edge_type, int64_t num_graph_edges,
                                           const int64_t *d_rel_edge_off,
                                           hifuse_layout layout, const hifuse_csr *out,
                                           void *d_ws, size_t ws_bytes, int32_t *d_status,
                                           hifuse_stream_t stream);

/* One-time graph preprocessing for the build: d_rel_edge_off[r] = first edge
 * id of relation r (lower bound of r in d_edge_type), r = 0..R, if
 * d_edge_type is sorted ascending (relation-major ids).  If it is not sorted
 * (or holds a relation id outside [0, R)), HIFUSE_ST_UNSORTED_TYPES is ORed
 * into *d_status and the offsets must not be used. */
hifuse_status hifuse_edge_type_offsets(const int32_t *d_edge_type, int64_t num_graph_edges,
                                       int num_rels, int64_t *d_rel_edge_off, int32_t *d_status,
                                       hifuse_stream_t stream);

/* A2+A3. Feature projection (readings C3, C4, C6, C7), one
 * grouped GEMM launch over groups {relation r} u {root type t}:
 *   Y[u]        = X_{s(r)}[y_src[u]] . W_rel[r]         u in relation r's rows
 *   R0[t,i]     = X_t[i] . W_root[t]                     i < n_dst[t] (if W_root)
 *   s_src[u,h]  = <Y[u, head h], att[r,0,head h]>        (if att, RGAT)
 *   s_dst[(r,i),h] = <(X_{t(r)}[i] W_rel[r])[head h], att[r,1,head h]>
 * X: fp32 [x_rows, K].  Row of (type t, local j) is type_src_off[t] + j, or,
 * when d_gather_ids != NULL, d_gather_ids[type_src_off[t] + j] (layer 0 reads
 * straight from the type-major feature store).
 * W_rel [R,K,D]; W_root [T,K,D] or NULL; att [R,2,D] or NULL.
 * Outputs: Y [U_max,D], R0 [sum_t n_dst[t], D] (if W_root), s_src [U_max,H],
 * s_dst [rows,H] (if att).  Workspace: hifuse_project_ws_bytes().
 * prec: FP32, TF32 or BF16 (see hifuse_prec). */
size_t hifuse_project_ws_bytes(const hifuse_layer_shape *shape, int K, int D, int heads);
/* hifuse_project for RGCN (no attention) with Y stored as bfloat16 (RN-even
 * rounding of the fp32 accumulator; SURVEY §8(f) NEXT(3) "BF16 storage of Y",
 * reading C25): d_Yb [U_max, D] bf16, 16-byte aligned; R0 fp32.  prec TF32
 * or BF16 (tcgen05 paths); FP32 -> HIFUSE_ERR_UNSUPPORTED.  The aggregation
 * then reads Y through hifuse_aggregate_features_cols_bf16 with d_col_x =
 * csr->col (Z[(r,i)] = sum_p w_p Y[col[p]]).  Workspace as hifuse_project. */
hifuse_status hifuse_project_y16(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                 hifuse_layout layout, hifuse_prec prec, int K, int D,
                                 const float *d_X, int64_t x_rows, const int32_t *d_gather_ids,
                                 const float *d_W_rel, const float *d_W_root, uint16_t *d_Yb,
                                 float *d_R0, void *d_ws, size_t ws_bytes,
                                 hifuse_stream_t stream);
hifuse_status hifuse_project(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                             hifuse_layout layout, hifuse_prec prec, int K, int D, int heads,
                             const float *d_X, int64_t x_rows, const int32_t *d_gather_ids,
                             const float *d_W_rel, const float *d_W_root, const float *d_att,
                             float *d_Y, float *d_R0, float *d_s_src, float *d_s_dst,
                             void *d_ws, size_t ws_bytes, hifuse_stream_t stream);

/* A4. Merged neighbour aggregation (Alg. 1): ONE
 * kernel for all relations.  For every merged row m = (r, i):
 *   SUM : Z[m] = sum_{p in row m} Y[col[p]]
 *   MEAN: Z[m] = SUM / |row m|                 (reading C1; IEEE division)
 *   GAT : per head h, alpha_p = softmax_{p in row m}(LeakyReLU_slope(
 *         s_src[col[p],h] + s_dst[m,h])); Z[m,head h] = sum alpha_p Y[col[p],head h]
 *         (readings C5, C6, C8); d_stats [rows, 2H] = (max, sum of exp) per
 *         (row, head), saved for the backward (reading C9).
 * Empty rows give Z = 0.  Relation-agnostic: only row_ptr/col are read. */
hifuse_status hifuse_aggregate_fwd(const hifuse_csr *csr, int64_t rows, hifuse_agg agg, int D,
                                   int heads, float slope, const float *d_Y,
                                   const float *d_s_src, const float *d_s_dst, float *d_Z,
                                   float *d_stats, hifuse_stream_t stream);

/* A4, GAT variant with the softmax ACROSS relations (SURVEY.md §8(f) NEXT(2),
 * DESIGN.md reading C5'; PAPER.md is silent on the softmax domain, line 123
 * leaves the fusion rule open).  For destination (t, i) and head h:
 *   alpha_p = softmax over the union of rows {(r, i) : t(r) = t} of
 *             LeakyReLU_slope(s_src[col[p],h] + s_dst[(r,i),h]),
 *   Z[(r,i), head h] = sum_{p in row (r,i)} alpha_p Y[col[p], head h],
 * so hifuse_semantic_fuse's sum over r is the attention-weighted sum over all
 * neighbours.  Still ONE kernel for all relations (one warp per destination,
 * walking its rows through the host-known rel_row_off).  d_stats [rows, 2H]
 * holds the destination's (max, sum of exp) in every one of its rows; empty
 * destinations give Z = 0, stats 0.  Arguments as hifuse_aggregate_fwd plus
 * the layer shape; errors: INVALID_ARG (null buffers), UNSUPPORTED (D not
 * 64/128, or D/H not a power of two >= 4), ALIGNMENT (Y, Z not 16-byte
 * aligned).  The backward is hifuse_aggregate_bwd with HIFUSE_AGG_GAT_XREL. */
hifuse_status hifuse_aggregate_fwd_xrel(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                        int D, int heads, float slope, const float *d_Y,
                                        const float *d_s_src, const float *d_s_dst, float *d_Z,
                                        float *d_stats, hifuse_stream_t stream);

/* A5. Semantic fusion (readings C2, C4, C10):
 *   H_t[i] = act(R0_t[i] + bias_t + sum_{r: t(r)=t} Z[rel_row_off[r] + i]).
 * Z [rows, D]; R0 [sum n_dst, D] or NULL; bias [T, D] or NULL; H [sum n_dst, D]
 * type-major (the next layer's X). */
hifuse_status hifuse_semantic_fuse(const hifuse_layer_shape *shape, int D, hifuse_act act,
                                   const float *d_Z, const float *d_R0, const float *d_bias,
                                   float *d_H, hifuse_stream_t stream);

/* A4 + A5 in one launch (RGCN sum / mean): hifuse_aggregate_fwd's Z rows
 * and hifuse_semantic_fuse's H, bit-identical to the two calls.  The warp
 * completing the last relation row (r, i) of destination (t, i) (a fenced
 * per-destination arrival counter) sums R0 + bias + the Z rows of t's
 * relations in relation order; destinations of a type no relation enters get
 * act(R0 + bias).  Arguments as for the two calls (Z is still written: the
 * rows of the other relations are read back from it).  Workspace:
 * hifuse_aggregate_fuse_ws_bytes() ints, ZEROED by the caller before the
 * first call; every call leaves it zeroed (CUDA-graph safe).  PAPER.md
 * lines 123 (fusion) and 246-262 (Alg. 1). */
size_t hifuse_aggregate_fuse_ws_bytes(const hifuse_layer_shape *shape);
hifuse_status hifuse_aggregate_fuse_fwd(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                        hifuse_agg agg, int D, hifuse_act act, const float *d_Y,
                                        const float *d_R0, const float *d_bias, float *d_Z,
                                        float *d_H, void *d_ws, size_t ws_bytes,
                                        hifuse_stream_t stream);

/* A6a. Fusion backward: G = dH * act'(H) (ReLU' = 1[H > 0]); G is dR0 and
 * the gradient of every Z row (r, i) (= G_{t(r)}[i]); dbias_t = sum_i G_t[i]
 * (fixed-order two-stage reduction).  dbias may be NULL.  Workspace:
 * hifuse_fuse_bwd_ws_bytes(). */
size_t hifuse_fuse_bwd_ws_bytes(const hifuse_layer_shape *shape, int D);
hifuse_status hifuse_semantic_fuse_bwd(const hifuse_layer_shape *shape, int D, hifuse_act act,
                                       const float *d_dH, const float *d_H, float *d_G,
                                       float *d_dbias, void *d_ws, size_t ws_bytes,
                                       hifuse_stream_t stream);
/* dbias_t = sum_i G_t[i] from a G formed by hifuse_semantic_fuse_bwd with
 * d_dbias = NULL: bit-identical to that call's dbias (same chunks, same
 * orders), so the critical path can form G alone and a parallel stream the
 * bias gradient.  Workspace: hifuse_fuse_bwd_ws_bytes(). */
hifuse_status hifuse_semantic_fuse_bwd_bias(const hifuse_layer_shape *shape, int D,
                                            const float *d_G, float *d_dbias, void *d_ws,
                                            size_t ws_bytes, hifuse_stream_t stream);

/* A5' / A6a'. HAN semantic-attention fusion (PAPER.md
 * line 123 leaves the fusion rule open; reading C22, HAN's semantic-level
 * attention [ext]).  Per relation r into type t, over the batch's n_t
 * destinations:
 *   w_r    = (1/n_t) sum_i q . tanh(Ws^T Z[rel_row_off[r] + i] + bs)
 *   beta_r = exp(w_r) / sum_{r': t(r')=t} exp(w_r')
 *   H_t[i] = act(R0_t[i] + bias_t + sum_r beta_r Z[rel_row_off[r] + i]).
 * d_Ws [D, A] row-major, d_bs [A], d_q [A]; A == D (64 or 128).  Outputs
 * d_beta [R] (kept for the backward), d_w [R] (nullable), d_H.  Workspace:
 * hifuse_sem_att_ws_bytes() (the same buffer serves the backward).
 * Backward: G = dH act'(H) (= dR0), dbias, and the per-merged-row gradient
 *   dZ[(r,i)] = beta_r G_t[i] + Ws (c_r q (.) (1 - tanh^2(a))),
 *   c_r = beta_r (dbeta_r - sum_{r'|t} beta_r' dbeta_r') / n_t,
 *   dbeta_r = sum_i <G_t[i], Z[(r,i)]>,  a = Ws^T Z[(r,i)] + bs,
 * plus dWs, dbs, dq (fixed-order reductions); dZ feeds
 * hifuse_aggregate_bwd_rows. */
size_t hifuse_sem_att_ws_bytes(const hifuse_layer_shape *shape, int D, int A);
hifuse_status hifuse_semantic_fuse_att(const hifuse_layer_shape *shape, int D, int A,
                                       hifuse_act act, const float *d_Z, const float *d_R0,
                                       const float *d_bias, const float *d_Ws,
                                       const float *d_bs, const float *d_q, float *d_beta,
                                       float *d_w, float *d_H, void *d_ws, size_t ws_bytes,
                                       hifuse_stream_t stream);
hifuse_status hifuse_semantic_fuse_att_bwd(const hifuse_layer_shape *shape, int D, int A,
                                           hifuse_act act, const float *d_dH, const float *d_H,
                                           const float *d_Z, const float *d_Ws,
                                           const float *d_bs, const float *d_q,
                                           const float *d_beta, float *d_G, float *d_dZ,
                                           float *d_dbias, float *d_dWs, float *d_dbs,
                                           float *d_dq, void *d_ws, size_t ws_bytes,
                                           hifuse_stream_t stream);

/* A6b. Aggregation backward: the transpose gather over the CSC.
 *   SUM/MEAN: dY[u] = sum_{q in col u} w(row_q) G[g(row_q)],  w = 1 or 1/|row|
 *   GAT: pass 1 (row-major) recomputes alpha from d_stats and forms
 *        dpre = alpha (dalpha - sum alpha dalpha) LeakyReLU', ds_dst[m,h] = sum dpre;
 *        pass 2 (CSC): dY[u,head h] = sum alpha G[g(row),head h], ds_src[u,h] = sum dpre.
 *   GAT_XREL: as GAT, but pass 1 runs per destination and sum alpha dalpha
 *        is taken over the destination's union of rows (the fused output).
 * g(r, i) = type_dst_off[t(r)] + i maps a merged row to its row of G.  dY
 * excludes the score-chain term (hifuse_project_bwd adds it).  Workspace:
 * hifuse_aggregate_bwd_ws_bytes() (GAT: 2 N H floats). */
size_t hifuse_aggregate_bwd_ws_bytes(const hifuse_layer_shape *shape, hifuse_agg agg, int heads);
hifuse_status hifuse_aggregate_bwd(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                   hifuse_agg agg, int D, int heads, float slope,
                                   const float *d_G, const float *d_Y, const float *d_s_src,
                                   const float *d_s_dst, const float *d_stats, float *d_dY,
                                   float *d_ds_src, float *d_ds_dst, void *d_ws, size_t ws_bytes,
                                   hifuse_stream_t stream);

/* Aggregation backward for a PER-MERGED-ROW gradient d_dZ [rows, D] (dL/dZ,
 * e.g. after HAN semantic-attention fusion, where the relations of a type get
 * different gradients: hifuse_semantic_fuse_att_bwd) instead of the
 * type-major G of hifuse_aggregate_bwd; otherwise identical.  d_att: NULL,
 * or (GAT kinds) the score chain is folded in as in
 * hifuse_aggregate_bwd_scored.  UNSUPPORTED for GAT_XREL. */
hifuse_status hifuse_aggregate_bwd_rows(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                        hifuse_agg agg, int D, int heads, float slope,
                                        const float *d_dZ, const float *d_Y,
                                        const float *d_s_src, const float *d_s_dst,
                                        const float *d_stats, const float *d_att, float *d_dY,
                                        float *d_ds_src, float *d_ds_dst, void *d_ws,
                                        size_t ws_bytes, hifuse_stream_t stream);

/* RGAT, score chain folded into the CSC pass: as hifuse_aggregate_bwd (GAT or
 * GAT_XREL) but d_dY receives dYt = dY + ds_src (x) att[r, 0] directly (the
 * term hifuse_project_bwd would otherwise add in place, same fp32 fma), so
 * the projection backward must then be hifuse_project_bwd_scored.  d_att
 * [R, 2, D] (16-byte aligned); INVALID_ARG for SUM/MEAN or NULL d_att. */
hifuse_status hifuse_aggregate_bwd_scored(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                          hifuse_agg agg, int D, int heads, float slope,
                                          const float *d_G, const float *d_Y,
                                          const float *d_s_src, const float *d_s_dst,
                                          const float *d_stats, const float *d_att, float *d_dY,
                                          float *d_ds_src, float *d_ds_dst, void *d_ws,
                                          size_t ws_bytes, hifuse_stream_t stream);

/* A6c. Projection backward, the adjoint of hifuse_project:
 *   dYt = dY + ds_src (x) att[r,0]             (score chain, RGAT; d_dY updated in place)
 *   dW_rel[r]  = sum_u X_row(u)^T dYt[u] (+ s_dst chain)   dW_root[t] = sum_i X_t[i]^T G_t[i]
 *   datt[r]    = (sum_u ds_src[u,h] Y[u,head h] | sum_i ds_dst v-chain)
 *   dX (optional, NULL for layer 0) = sum of dYt W_r^T + G W_root^T + ds_dst-chain.
 * d_dW_rel = d_dW_root = NULL (d_dX required): the input gradient alone
 * (RGAT: the dgrad plus the s_dst chain's dX term, with the W a_dst fold on a
 * parallel branch; only through hifuse_project_bwd_scored, whose dY already
 * holds dYt, so that the score chain is applied once; d_datt may be NULL);
 * a second call with d_dX = NULL forms the weight (and attention) gradients,
 * so the caller can run it on a parallel stream while the next layer's
 * backward proceeds.  Both forms are bit-identical to the combined call.  Fixed-order chunked reductions (deterministic).  Workspace:
 * hifuse_project_bwd_ws_bytes(). */
size_t hifuse_project_bwd_ws_bytes(const hifuse_layer_shape *shape, int K, int D, int heads);
hifuse_status hifuse_project_bwd(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                 hifuse_layout layout, hifuse_prec prec, int K, int D, int heads,
                                 const float *d_X, int64_t x_rows, const int32_t *d_gather_ids,
                                 const float *d_W_rel, const float *d_W_root, const float *d_att,
                                 const float *d_Y, float *d_dY, const float *d_G,
                                 const float *d_ds_src, const float *d_ds_dst, float *d_dX,
                                 float *d_dW_rel, float *d_dW_root, float *d_datt,
                                 void *d_ws, size_t ws_bytes, hifuse_stream_t stream);

/* Aggregate-first RGCN input layer.
 * The RGCN message is linear, so Z_r = A_r (X W_r) = (A_r X) W_r exactly: the
 * paper's stages 2-3 (projection, aggregation) may
 * run in the other order.  For the input layer this projects rho aggregated
 * rows instead of U compact source rows and needs no transpose SpMM.
 *
 * hifuse_aggregate_features_fwd: Alg. 1's merged Aggregate over the RAW
 *   features, Xagg[(r,i)] = sum (SUM) or mean (MEAN) over the row's edges of
 *   X[x(e)], x(e) = gather_ids[type_src_off[s(r)] + src_local(e)] (gather_ids
 *   NULL: identity).  Xagg [rows, K]; empty rows 0.  Same kernel as A4.
 *   Workspace: hifuse_aggregate_features_ws_bytes() (N ints).
 * hifuse_project_aggregated: Z[(r,i)] = Xagg[(r,i)] W_r (per-relation groups
 *   over rel_row_off), R0_t = X_t[dst prefix] W_root_t (X gathered through
 *   gather_ids).  tcgen05 TF32 only.
 * hifuse_project_aggregated_bwd: dW_r = sum_i Xagg[(r,i)]^T G_t(r)[i],
 *   dW_root_t = sum_i X_t[i]^T G_t[i] (G from hifuse_semantic_fuse_bwd);
 *   no dX (input layer).  Fixed-order chunk reduction.  Workspace:
 *   hifuse_project_aggregated_bwd_ws_bytes(). */
size_t hifuse_aggregate_features_ws_bytes(const hifuse_layer_shape *shape);
hifuse_status hifuse_aggregate_features_fwd(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                            hifuse_agg agg, int K, const float *d_X,
                                            int64_t x_rows, const int32_t *d_gather_ids,
                                            float *d_Xagg, void *d_ws, size_t ws_bytes,
                                            hifuse_stream_t stream);
/* NEXT(3) fused fusion GEMM of the aggregate-first RGCN input layer (SURVEY.md
 * §8(f) row 3): hifuse_project_aggregated and
 * hifuse_semantic_fuse as ONE tcgen05 TF32 GEMM per destination type,
 *   H_t[i] = act([X_t[i] | Xagg[rel_row_off[r1] + i] | ...] . [W_root,t; W_r1; ...] + b_t),
 * K = (1 + R_in(t)) K_in (relations r into t in ascending id; the root term
 * when d_W_root != NULL, reading X through d_gather_ids like
 * hifuse_project_aggregated), bias and activation in the epilogue; writes H
 * [sum_t n_dst(t), D] directly (no Z / R0).  Same values as the two calls up
 * to the fp32 summation order.  The backward is unchanged
 * (hifuse_semantic_fuse_bwd + hifuse_project_aggregated_bwd). */
hifuse_status hifuse_project_fuse_aggregated(const hifuse_layer_shape *shape,
                                            const hifuse_csr *csr, hifuse_prec prec, int K, int D,
                                            hifuse_act act, const float *d_Xagg,
                                            const float *d_X, int64_t x_rows,
                                            const int32_t *d_gather_ids, const float *d_W_rel,
                                            const float *d_W_root, const float *d_bias,
                                            float *d_H, hifuse_stream_t stream);

/* NEXT(3) BF16 storage of the input features (byte
 * diet): hifuse_aggregate_features_cols over a BF16 feature store d_Xb
 * (bfloat16 [x_rows, K], RN-even rounded by the caller), fp32 accumulation in
 * the same order, fp32 Xagg out -- half the bytes of the layer's dominant
 * read.  d_Xdst (nullable, fp32 [sum_t n_src(t), K]): the layer's destination
 * rows (the root term's X rows) converted to fp32 at rows type_src_off[t] +
 * i, i < n_dst(t) (other rows untouched), for the tcgen05 GEMMs
 * (hifuse_project_fuse_aggregated / hifuse_project_aggregated_bwd with
 * d_X = d_Xdst, d_gather_ids = NULL).  Same launch. */
hifuse_status hifuse_aggregate_features_cols_bf16(const hifuse_layer_shape *shape,
                                                  const hifuse_csr *csr, hifuse_agg agg, int K,
                                                  const void *d_Xb, int64_t x_rows,
                                                  const int32_t *d_col_x,
                                                  const int32_t *d_gather_ids, float *d_Xagg,
                                                  float *d_Xdst, hifuse_stream_t stream);

/* The two halves of hifuse_aggregate_features_fwd, so the first can run with
 * the semantic-graph build (off the critical path):
 *   hifuse_feature_cols: d_col_x [N] = the feature-store row x(e) of every
 *     CSR position (gather_ids NULL: identity), from a Y-numbered or an
 *     X-row-mode build (an X-row build with x_gather already wrote exactly
 *     this map into col: use col directly);
 *   hifuse_aggregate_features_cols: the aggregation over X rows d_col_x. */
hifuse_status hifuse_feature_cols(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                  const int32_t *d_gather_ids, int32_t *d_col_x,
                                  hifuse_stream_t stream);
hifuse_status hifuse_aggregate_features_cols(const hifuse_layer_shape *shape,
                                             const hifuse_csr *csr, hifuse_agg agg, int K,
                                             const float *d_X, int64_t x_rows,
                                             const int32_t *d_col_x, float *d_Xagg,
                                             hifuse_stream_t stream);
hifuse_status hifuse_project_aggregated(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                        hifuse_prec prec, int K, int D, const float *d_Xagg,
                                        const float *d_X, int64_t x_rows,
                                        const int32_t *d_gather_ids, const float *d_W_rel,
                                        const float *d_W_root, float *d_Z, float *d_R0,
                                        hifuse_stream_t stream);
size_t hifuse_project_aggregated_bwd_ws_bytes(const hifuse_layer_shape *shape, int K, int D);
hifuse_status hifuse_project_aggregated_bwd(const hifuse_layer_shape *shape,
                                            const hifuse_csr *csr, hifuse_prec prec, int K, int D,
                                            const float *d_Xagg, const float *d_X, int64_t x_rows,
                                            const int32_t *d_gather_ids, const float *d_G,
                                            float *d_dW_rel, float *d_dW_root, void *d_ws,
                                            size_t ws_bytes, hifuse_stream_t stream);

/* Training-step helpers outside the paper's four stages:
 * linear classifier + mean softmax cross-entropy on the seed rows, its
 * gradients, and the SGD update p -= lr * g over a flat parameter buffer.
 *   logits = Hs Wc + bc  (Hs [B, D] rows of d_H starting at row h_row0)
 *   loss   = mean_b (logsumexp(logits_b) - logits_b[label_b])    -> d_loss [1]
 *   dH (rows h_row0.. of d_dH; all other rows zeroed), dWc [D,C], dbc [C].
 * Three kernels (logits, row softmax, gradients; 3xTF32 mma.sync, fp32-level
 * accuracy).  d_dWc = d_dbc = NULL defers the weight gradient to hifuse_linear_xent_wgrad (same
 * workspace), so a caller can run it on a parallel branch next to the
 * backward of the HGNN layers. */
size_t hifuse_xent_ws_bytes(int B, int D, int C);
hifuse_status hifuse_linear_xent(int B, int D, int C, const float *d_H, int64_t h_rows,
                                 int64_t h_row0, const int32_t *d_labels, const float *d_Wc,
                                 const float *d_bc, float *d_loss, float *d_dH, float *d_dWc,
                                 float *d_dbc, void *d_ws, size_t ws_bytes, int32_t *d_status,
                                 hifuse_stream_t stream);
/* d_status (nullable): a label outside [0, C) ORs HIFUSE_ST_BAD_LABEL; that
 * row contributes no loss and no gradient (the loss is still divided by B).
 * dWc = Hs^T dlog, dbc = column sums of dlog from the dlog a preceding
 * hifuse_linear_xent (d_dWc = NULL) left in d_ws. */
hifuse_status hifuse_linear_xent_wgrad(int B, int D, int C, const float *d_H, int64_t h_rows,
                                       int64_t h_row0, float *d_dWc, float *d_dbc, void *d_ws,
                                       size_t ws_bytes, hifuse_stream_t stream);
hifuse_status hifuse_sgd(float *d_param, const float *d_grad, int64_t n, float lr, float grad_scale,
                         hifuse_stream_t stream);

/* hifuse_project_bwd for a d_dY that already holds dYt (produced by
 * hifuse_aggregate_bwd_scored): identical except that the in-place score-chain
 * update of d_dY is skipped.  d_att required. */
hifuse_status hifuse_project_bwd_scored(const hifuse_layer_shape *shape, const hifuse_csr *csr,
                                        hifuse_layout layout, hifuse_prec prec, int K, int D,
                                        int heads, const float *d_X, int64_t x_rows,
                                        const int32_t *d_gather_ids, const float *d_W_rel,
                                        const float *d_W_root, const float *d_att,
                                        const float *d_Y, float *d_dY, const float *d_G,
                                        const float *d_ds_src, const float *d_ds_dst,
                                        float *d_dX, float *d_dW_rel, float *d_dW_root,
                                        float *d_datt, void *d_ws, size_t ws_bytes,
                                        hifuse_stream_t stream);

/* ------------------------------------------------------------------------
 * NEXT(1): GPU neighbour sampler.  PAPER.md Fig. 2 step (1)
 * ("mini-batches are sampled from the original graph", line 156) and SPEC.md
 * sample_batch: each (vertex, relation) pair of a layer's
 * destinations contributes min(deg, fanout) of its in-edges, chosen uniformly
 * WITHOUT replacement; message-flow block convention (reading C12): per type
 * the layer's destinations are the first n_dst of its sources, new sources
 * follow in ascending vertex id.  Randomness: Floyd's subset algorithm driven
 * by a counter-based splitmix64 hash of (hop key, relation, vertex, j), so a
 * batch is a pure function of (graph, seeds, fanout, key) -- any rank, any
 * order.  Edge order inside a block: destination (type-major,
 * local id), then relation ascending, then in-list position ascending.
 * Everything runs on the device; capacities are host-known (graph-capturable);
 * the data-dependent sizes land in hifuse_block.counts.
 * ------------------------------------------------------------------------ */
typedef struct {                  /* in-adjacency of the whole graph, per relation */
  int32_t num_types, num_rels;
  const int32_t *rel_src_type_h, *rel_dst_type_h;   /* [R] host */
  const int64_t *type_count_h;    /* [T] host: |V_t| */
  const int64_t *in_ptr_off_h;    /* [R] host: relation r's block of d_in_ptr starts here */
  const int64_t *d_in_ptr;        /* device [sum_r (|V_t(r)| + 1)]: for vertex v of type
                                   * t(r), its in-edges are positions
                                   * [d_in_ptr[off_r + v], d_in_ptr[off_r + v + 1]) of: */
  const int32_t *d_in_src;        /* device [E]: source vertex (id within its type)    */
  const int64_t *d_in_eid;        /* device [E]: global edge id (EdgeType index)       */
} hifuse_graph_csc;

typedef struct {                  /* one sampled layer block (device, caller-allocated) */
  int32_t *src_local, *dst_local; /* [edge_cap] */
  int64_t *edge_id;               /* [edge_cap] */
  int32_t *src_gid;               /* [src_cap] type-major source vertices (ids within type);
                                   * the first n_dst(t) of type t are the destinations */
  int32_t *counts;                /* [2T + 1]: n_src[T], n_dst[T], N */
  int32_t *gather_ids;            /* [src_cap] or NULL: type_off(t) + src_gid, type_off =
                                   * prefix of type_count_h (type-major feature store) */
} hifuse_block;

/* Host-only: per layer (outer first) the edge / source capacities the caller
 * allocates, the workspace bytes, and the sampler state ints (2 sum_t |V_t|,
 * zeroed once by the caller before the first call). */
hifuse_status hifuse_sample_caps(const hifuse_graph_csc *g, int num_layers,
                                 const int32_t *fanout_h /* [L], outer layer first */,
                                 int64_t num_seeds, int64_t *edge_cap_h /* [L] */,
                                 int64_t *src_cap_h /* [L] */, size_t *ws_bytes,
                                 int64_t *state_ints);
/* Samples num_layers blocks around d_seeds (ids within target_type) into
 * out[L] (outer layer first).  key: 64-bit stream key of this batch (e.g. a
 * splitmix64 of (seed, epoch, batch)); hop h uses mix(key ^ (0x1000 + h)).
 * d_ctl: NULL, or device uint64 [2] = {key, stamp}: key and stamp are then
 * read from device memory instead of the arguments, so one captured CUDA graph
 * of the sampler serves every batch (write the next {key, stamp}, replay).
 * d_state: sampler state (see caps), stamps [stamp, stamp + L) must not have
 * been used since it was zeroed (stamp >= 1).  d_status: HIFUSE_ST_BAD_DST is
 * ORed for a seed out of range (it is dropped).  Errors: INVALID_ARG (null
 * pointers, fanout < 1 or > 64, target_type out of range), WORKSPACE. */
hifuse_status hifuse_sample_blocks(const hifuse_graph_csc *g, int num_layers,
                                   const int32_t *fanout_h, const int32_t *d_seeds,
                                   int64_t num_seeds, int32_t target_type, uint64_t key,
                                   const uint64_t *d_ctl, int32_t stamp, hifuse_block *out,
                                   int32_t *d_state,
                                   void *d_ws, size_t ws_bytes, int32_t *d_status,
                                   hifuse_stream_t stream);

/* Padded (capacity) layout of the same sampler, so that ONE captured CUDA
 * graph of sampler + build + training step serves every batch (the step's
 * host shapes become the capacities; Fig. 6, with
 * sampling inside the pipelined loop).  src_cap_h [L*T] (outer layer first,
 * row l): sources of type t in layer l occupy slots [off_l(t), off_l(t) +
 * src_cap_h[l*T+t]) of src_gid / gather_ids, off_l = prefix of the row; the
 * layer's destinations (layer l+1's padded sources, or the seeds) are the
 * first slots of each type, so src_cap_h[l*T+t] >= src_cap_h[(l+1)*T+t].
 * Slots past the sampled sources hold src_gid -1 (gather id: the type's
 * first feature row); padded destinations (src_gid -1) are not sampled.
 * Edge positions [N, edge_pad_h[l]) hold null edges (edge_id -1, ids 0),
 * which the build drops silently.  counts: n_src[t] = padded destinations +
 * sampled new sources, n_dst[t] = padded destinations, N = sampled edges; a
 * block past its capacities ORs HIFUSE_ST_OVERFLOW into d_status (its layout
 * is then invalid: the caller re-samples it in the compact layout).  Output
 * buffers as for hifuse_sample_blocks (worst-case capacities).  Errors:
 * INVALID_ARG also for capacities that break the rules above or exceed the
 * worst-case capacities of hifuse_sample_caps. */
hifuse_status hifuse_sample_blocks_padded(const hifuse_graph_csc *g, int num_layers,
                                          const int32_t *fanout_h, const int32_t *d_seeds,
                                          int64_t num_seeds, int32_t target_type, uint64_t key,
                                          const uint64_t *d_ctl, int32_t stamp,
                                          const int64_t *src_cap_h /* [L*T] */,
                                          const int64_t *edge_pad_h /* [L] */,
                                          hifuse_block *out, int32_t *d_state, void *d_ws,
                                          size_t ws_bytes, int32_t *d_status,
                                          hifuse_stream_t stream);

/* Per-stream fork/join resources (common.cu).  A call that runs independent
 * kernels concurrently (the dgrad || wgrad of hifuse_project_bwd, the two
 * RGAT attention chains, the RGAT destination scores || the projection)
 * forks them onto auxiliary streams owned by the caller's stream `stream`
 * (created on first use; under CUDA-graph capture the fork becomes a parallel
 * graph branch).  hifuse_stream_attach creates them ahead of time -- call it
 * outside capture for every stream that will later be captured;
 * HIFUSE_ERR_INVALID_ARG if `stream` is capturing.  hifuse_stream_release
 * destroys them (synchronises the auxiliary streams; the caller guarantees no
 * call on `stream` is in flight or later replayed from a graph).  If the
 * resources cannot be created, branches run serially on `stream`.  No
 * arithmetic; PAPER.md has no counterpart (a B200 scheduling detail, DESIGN
 * §9 "Backward off the critical path"). */
hifuse_status hifuse_stream_attach(hifuse_stream_t stream);
hifuse_status hifuse_stream_release(hifuse_stream_t stream);

/* NEXT(4) feature-sharded data parallelism (PAPER.md
 * line 219 "a large heterogeneous graph can be partitioned into several
 * subgraphs", line 404).  Rank k keeps rows [bounds[k], bounds[k+1]) of the
 * type-major feature store; before A2 a batch's layer-0 rows are fetched from
 * their owners with one all-to-all of ids and one of rows (shard.py).
 * hifuse_shard_plan: stable counting sort of d_ids [n] (global rows) by owner:
 *   d_counts [W] per-owner counts, d_order [n] batch positions grouped by
 *   owner (batch order inside an owner); W <= 64, d_bounds int64 [W+1]
 *   ascending.  Ids outside [bounds[0], bounds[W]) set HIFUSE_ST_BAD_EDGE_ID
 *   and are left out.
 * hifuse_gather_words: dst[i] = src[idx[i] - base] for rows of `words`
 *   4-byte words (16-byte vectors when words % 4 == 0 and both aligned).
 * hifuse_scatter_words: dst[idx[i]] = src[i] (rows of `words` words). */
hifuse_status hifuse_shard_plan(const int32_t *d_ids, int64_t n, const int64_t *d_bounds, int W,
                                int32_t *d_counts, int32_t *d_order, int32_t *d_status,
                                hifuse_stream_t stream);
hifuse_status hifuse_gather_words(const void *d_src, const int32_t *d_idx, int64_t n, int words,
                                  int64_t base, void *d_dst, hifuse_stream_t stream);
hifuse_status hifuse_scatter_words(const void *d_src, const int32_t *d_idx, int64_t n, int words,
                                   void *d_dst, hifuse_stream_t stream);

/* Tests / debugging: copies *d_status to *out_h and synchronises `stream`. */
hifuse_status hifuse_read_status(const int32_t *d_status, hifuse_stream_t stream, int32_t *out_h);
const char *hifuse_status_string(hifuse_status s);
/* Number of kernels launched by this process so far (host counter). */
int64_t hifuse_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* HIFUSE_H */

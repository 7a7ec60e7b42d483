/*
 * hifuse_oracle.c -- plain, slow, obviously-correct CPU oracle of the HiFuse
 * hot path (arXiv 2408.08490).  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  It shares no code, header, table or helper with the CUDA
 * library under paper_2408_08490_b200/csrc/.
 *
 * Every function follows one passage of PAPER.md (the "P:Lnn" line numbers are
 * those of /root/reference/PAPER.md) or, where the paper is silent, one reading
 * of DESIGN.md §Readings (C1..C21).  Arithmetic is fp64 on fp64 inputs; loops
 * go relation by relation, the way Alg. 1 and Alg. 2 are written.
 *
 * Pins: tests/test_oracle_*.py (brute-force dense adjacency, library special
 * cases, hand examples from SPEC.md, finite differences, adjoint identities).
 *
 * Threads (OpenMP, oracle_set_threads; default 1): only loops whose
 * iterations write disjoint outputs run in parallel, and every output element
 * is accumulated in the same order as the serial loop, so results are
 * bit-identical for any thread count (tests/test_oracle_threads.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* number of OpenMP threads of the parallel loops below (1: serial) */
void oracle_set_threads(int n)
{
#ifdef _OPENMP
    omp_set_num_threads(n > 0 ? n : 1);
#else
    (void)n;
#endif
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

#define ST_BAD_EDGE_ID 1   /* edge_id >= E_graph or < 0            */
#define ST_BAD_REL     2   /* edge_type[edge_id] not in [0, R)     */
#define ST_BAD_SRC     4   /* src local id >= n_src(s(r))          */
#define ST_BAD_DST     8   /* dst local id >= n_dst(t(r))          */

/* ------------------------------------------------------------------------ */
/* O1. Semantic graph build = Alg. 2 + bucketing into rows.     */
/* ------------------------------------------------------------------------ */
/*
 * Alg. 2: EdgeTypeLayer <- IndexSelect(EdgeType, EdgeID[i]).
 * Alg. 2: for each relation j, mask <- compare(j, EdgeTypeLayer),
 *   TempEdgeIndex <- IndexSelect(EdgeIndex[i], mask)  (column order kept).
 * Then (reading C2, C14): relation j's edges are bucketed per destination
 * vertex, rows ordered (relation ascending, dst ascending), edges inside a row
 * in ascending original column; the merged projected matrix Y holds, per
 * relation, one row per distinct source vertex, ascending (layout "compact",
 * reading C3); col[p] is the Y row of the edge at CSR position p; the CSC
 * lists, per Y row, the CSR positions that read it, ascending.
 * Invalid edges (status bits) are dropped; unused tails are set to -1.
 * Edge id -1 is a null edge (capacity padding, reading C26): it is
 * dropped without a status bit.
 */
int oracle_build(int T, int R, const int32_t *rel_src, const int32_t *rel_dst,
                 const int32_t *n_src, const int32_t *n_dst,
                 int64_t N, const int32_t *src, const int32_t *dst, const int64_t *eid,
                 const int32_t *edge_type, int64_t E,
                 int32_t *rel_row_off, int32_t *row_ptr, int32_t *col, int32_t *eperm,
                 int32_t *rel_y_off, int32_t *y_src, int32_t *col_ptr,
                 int32_t *csc_pos, int32_t *csc_row, int32_t *slot_y, int32_t *U_out)
{
    int status = 0;
    (void)T;
    /* line 316: EdgeTypeLayer */
    int32_t *etl = (int32_t *)malloc(sizeof(int32_t) * (N > 0 ? N : 1));
    for (int64_t e = 0; e < N; e++) {
        etl[e] = -1;
        if (eid[e] == -1) continue;        /* null (padding) edge: dropped, no status (C26) */
        if (eid[e] < 0 || eid[e] >= E) { status |= ST_BAD_EDGE_ID; continue; }
        int32_t r = edge_type[eid[e]];
        if (r < 0 || r >= R) { status |= ST_BAD_REL; continue; }
        if (src[e] < 0 || src[e] >= n_src[rel_src[r]]) { status |= ST_BAD_SRC; continue; }
        if (dst[e] < 0 || dst[e] >= n_dst[rel_dst[r]]) { status |= ST_BAD_DST; continue; }
        etl[e] = r;
    }
    /* row offsets of each relation's destination block */
    int64_t rows = 0;
    for (int r = 0; r < R; r++) { rel_row_off[r] = (int32_t)rows; rows += n_dst[rel_dst[r]]; }
    rel_row_off[R] = (int32_t)rows;
    int64_t S = 0;
    int64_t *slot_off = (int64_t *)malloc(sizeof(int64_t) * (R + 1));
    for (int r = 0; r < R; r++) { slot_off[r] = S; S += n_src[rel_src[r]]; }
    slot_off[R] = S;
    for (int64_t s = 0; s < S; s++) slot_y[s] = -1;

    /* per-row edge lists, filled relation by relation (lines 317-321) */
    int64_t *row_cnt = (int64_t *)calloc((size_t)rows + 1, sizeof(int64_t));
    int64_t p = 0;
    int32_t U = 0;
    for (int r = 0; r < R; r++) {
        /* mask <- compare(r, EdgeTypeLayer); selected columns in order */
        int64_t nsel = 0;
        for (int64_t e = 0; e < N; e++) if (etl[e] == r) nsel++;
        int64_t *sel = (int64_t *)malloc(sizeof(int64_t) * (nsel > 0 ? nsel : 1));
        nsel = 0;
        for (int64_t e = 0; e < N; e++) if (etl[e] == r) sel[nsel++] = e;
        /* compact Y rows of relation r: sorted unique sources */
        rel_y_off[r] = U;
        int32_t ns = n_src[rel_src[r]];
        for (int64_t k = 0; k < nsel; k++) slot_y[slot_off[r] + src[sel[k]]] = 0;
        for (int32_t j = 0; j < ns; j++)
            if (slot_y[slot_off[r] + j] == 0) { y_src[U] = j; slot_y[slot_off[r] + j] = U; U++; }
            else slot_y[slot_off[r] + j] = -1;
        /* bucket the selected edges per destination, column order kept:
         * count per destination, then place in selection order (stable). */
        int32_t nd = n_dst[rel_dst[r]];
        for (int64_t k = 0; k < nsel; k++) row_cnt[rel_row_off[r] + dst[sel[k]]]++;
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (nd > 0 ? nd : 1));
        for (int32_t i = 0; i < nd; i++) {
            int64_t row = rel_row_off[r] + i;
            row_ptr[row] = (int32_t)p;
            fill[i] = p;
            p += row_cnt[row];
        }
        for (int64_t k = 0; k < nsel; k++) {
            int64_t e = sel[k];
            int64_t q = fill[dst[e]]++;
            eperm[q] = (int32_t)e;
            col[q] = slot_y[slot_off[r] + src[e]];
        }
        free(fill);
        free(sel);
    }
    rel_y_off[R] = U;
    row_ptr[rows] = (int32_t)p;
    for (int64_t q = p; q < N; q++) { col[q] = -1; eperm[q] = -1; csc_pos[q] = -1; csc_row[q] = -1; }
    /* merged row of every CSR position */
    int32_t *row_of = (int32_t *)malloc(sizeof(int32_t) * (p > 0 ? p : 1));
    for (int64_t row = 0; row < rows; row++)
        for (int64_t q = row_ptr[row]; q < row_ptr[row + 1]; q++) row_of[q] = (int32_t)row;
    /* CSC over Y rows: positions ascending inside each column (count per
     * column, then place positions in ascending order: stable). */
    int64_t *ccnt = (int64_t *)calloc((size_t)U + 1, sizeof(int64_t));
    for (int64_t q = 0; q < p; q++) ccnt[col[q]]++;
    int64_t c = 0;
    for (int32_t u = 0; u < U; u++) { col_ptr[u] = (int32_t)c; c += ccnt[u]; ccnt[u] = col_ptr[u]; }
    for (int64_t q = 0; q < p; q++) {
        int64_t w = ccnt[col[q]]++;
        csc_pos[w] = (int32_t)q;
        csc_row[w] = row_of[q];
    }
    free(ccnt);
    col_ptr[U] = (int32_t)c;
    *U_out = U;
    free(row_of); free(row_cnt); free(slot_off); free(etl);
    return status;
}

/* ------------------------------------------------------------------------ */
/* O2. Feature projection ("transformed using an MLP"), reading C3: */
/* per-relation weights W_r [K,D] on the relation's source rows, a root     */
/* weight W_root,t per destination type (C4); RGAT scores (C6, C7).         */
/* ------------------------------------------------------------------------ */
static const double *xrow(const double *X, int K, const int32_t *gather_ids,
                          const int64_t *type_src_off, int t, int32_t j)
{
    int64_t r = type_src_off[t] + j;
    if (gather_ids) r = gather_ids[r];
    return X + r * (int64_t)K;
}

void oracle_project(int T, int R, const int32_t *rel_src, const int32_t *rel_dst,
                    const int32_t *n_src, const int32_t *n_dst,
                    int K, int D, int H,
                    const double *X, const int32_t *gather_ids,
                    const int32_t *rel_y_off, const int32_t *y_src,
                    const double *W_rel, const double *W_root, const double *att,
                    double *Y, double *R0, double *s_src, double *s_dst)
{
    int64_t *tso = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    int64_t *tdo = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    tso[0] = tdo[0] = 0;
    for (int t = 0; t < T; t++) { tso[t + 1] = tso[t] + n_src[t]; tdo[t + 1] = tdo[t] + n_dst[t]; }
    int dh = D / H;
    /* Y[(r,j)] = X_{s(r)}[j] . W_r */
    for (int r = 0; r < R; r++) {
        const double *W = W_rel + (int64_t)r * K * D;
        #pragma omp parallel for schedule(static)
        for (int32_t u = rel_y_off[r]; u < rel_y_off[r + 1]; u++) {
            const double *x = xrow(X, K, gather_ids, tso, rel_src[r], y_src[u]);
            double *y = Y + (int64_t)u * D;
            for (int d = 0; d < D; d++) y[d] = 0.0;
            for (int k = 0; k < K; k++)
                for (int d = 0; d < D; d++) y[d] += x[k] * W[(int64_t)k * D + d];
            if (att) {   /* s_src[u,h] = <Y[u, head h], a_src^{r,h}> */
                const double *a_src = att + (int64_t)r * 2 * D;
                for (int h = 0; h < H; h++) {
                    double s = 0.0;
                    for (int c = 0; c < dh; c++) s += y[h * dh + c] * a_src[h * dh + c];
                    s_src[(int64_t)u * H + h] = s;
                }
            }
        }
    }
    /* R0_t[i] = X_t[i] . W_root,t  (destination prefix only) */
    if (W_root) {
        for (int t = 0; t < T; t++) {
            const double *W = W_root + (int64_t)t * K * D;
            #pragma omp parallel for schedule(static)
            for (int32_t i = 0; i < n_dst[t]; i++) {
                const double *x = xrow(X, K, gather_ids, tso, t, i);
                double *o = R0 + (tdo[t] + i) * (int64_t)D;
                for (int d = 0; d < D; d++) o[d] = 0.0;
                for (int k = 0; k < K; k++)
                    for (int d = 0; d < D; d++) o[d] += x[k] * W[(int64_t)k * D + d];
            }
        }
    }
    /* s_dst[(r,i),h] = <(X_{t(r)}[i] W_r)[head h], a_dst^{r,h}>  (reading C7) */
    if (att) {
        int64_t row0 = 0;
        for (int r = 0; r < R; r++) {
            const double *W = W_rel + (int64_t)r * K * D;
            const double *a_dst = att + (int64_t)r * 2 * D + D;
            int t = rel_dst[r];
            #pragma omp parallel
            {
                double *hv = (double *)malloc(sizeof(double) * D);
                #pragma omp for schedule(static)
                for (int32_t i = 0; i < n_dst[t]; i++) {
                    int64_t row = row0 + i;
                    const double *x = xrow(X, K, gather_ids, tso, t, i);
                    for (int d = 0; d < D; d++) hv[d] = 0.0;
                    for (int k = 0; k < K; k++)
                        for (int d = 0; d < D; d++) hv[d] += x[k] * W[(int64_t)k * D + d];
                    for (int h = 0; h < H; h++) {
                        double s = 0.0;
                        for (int c = 0; c < dh; c++) s += hv[h * dh + c] * a_dst[h * dh + c];
                        s_dst[row * H + h] = s;
                    }
                }
                free(hv);
            }
            row0 += n_dst[t];
        }
    }
    free(tso); free(tdo);
}

/* ------------------------------------------------------------------------ */
/* O3. Neighbor aggregation with merging = Alg. 1.            */
/* For each semantic graph i: Features <- IndexSelect(x[SrcType[i]],         */
/* SrcIndex[i]) (line 254); DstIndex appended (line 256); after the loop one */
/* Aggregate(FeatureCat, DstIndexCat) (line 260) whose segments are the      */
/* (relation, destination) pairs (reading C2).  agg: 0 sum, 1 mean (C1),     */
/* 2 GAT edge-softmax within (relation, destination) (C5, C6, C8), 3 GAT     */
/* edge-softmax across the relations of a destination (gat_xrel_fwd).        */
/* Edges are taken from the block itself (Alg. 2 selection, line 318), the   */
/* Y row of (r, src) from the compact layout (rel_y_off, y_src).             */
/* ------------------------------------------------------------------------ */
static int32_t yrow_of(const int32_t *rel_y_off, const int32_t *y_src, int r, int32_t j)
{
    int32_t lo = rel_y_off[r], hi = rel_y_off[r + 1];   /* y_src ascending in [lo, hi) */
    while (lo < hi) {
        int32_t mid = lo + (hi - lo) / 2;
        if (y_src[mid] < j) lo = mid + 1; else hi = mid;
    }
    if (lo < rel_y_off[r + 1] && y_src[lo] == j) return lo;
    /* a valid edge whose source is missing from y_src: the caller passed an
     * inconsistent (rel_y_off, y_src); fail loudly, never index Y[-1] */
    fprintf(stderr, "oracle: yrow_of: source %d of relation %d not in y_src\n", (int)j, r);
    abort();
}

static int valid_edge(int R, const int32_t *rel_src, const int32_t *rel_dst,
                      const int32_t *n_src, const int32_t *n_dst, int64_t e,
                      const int32_t *src, const int32_t *dst, const int64_t *eid,
                      const int32_t *edge_type, int64_t E)
{
    if (eid[e] < 0 || eid[e] >= E) return -1;
    int32_t r = edge_type[eid[e]];
    if (r < 0 || r >= R) return -1;
    if (src[e] < 0 || src[e] >= n_src[rel_src[r]]) return -1;
    if (dst[e] < 0 || dst[e] >= n_dst[rel_dst[r]]) return -1;
    return r;
}

/* Relation r's selected edges bucketed per destination, column order kept
 * (Alg. 2 selection, line 318-319, then a stable bucket by DstIndex). */
static void relation_rows(int R, const int32_t *rel_src, const int32_t *rel_dst,
                          const int32_t *n_src, const int32_t *n_dst, int r,
                          int64_t N, const int32_t *src, const int32_t *dst, const int64_t *eid,
                          const int32_t *edge_type, int64_t E,
                          int64_t **ptr_out, int64_t **list_out)
{
    int32_t nd = n_dst[rel_dst[r]];
    int64_t *ptr = (int64_t *)calloc((size_t)nd + 1, sizeof(int64_t));
    int64_t n = 0;
    for (int64_t e = 0; e < N; e++)
        if (valid_edge(R, rel_src, rel_dst, n_src, n_dst, e, src, dst, eid, edge_type, E) == r) {
            ptr[dst[e] + 1]++; n++;
        }
    for (int32_t i = 0; i < nd; i++) ptr[i + 1] += ptr[i];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (nd > 0 ? nd : 1));
    for (int32_t i = 0; i < nd; i++) fill[i] = ptr[i];
    int64_t *list = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    for (int64_t e = 0; e < N; e++)
        if (valid_edge(R, rel_src, rel_dst, n_src, n_dst, e, src, dst, eid, edge_type, E) == r)
            list[fill[dst[e]]++] = e;
    free(fill);
    *ptr_out = ptr; *list_out = list;
}

static double leaky(double x, double slope) { return x > 0 ? x : slope * x; }

/* Attention logit of an edge from its source score ss and destination score
 * sd: agg 2/3 additive GAT (reading C6) LeakyReLU(ss + sd); agg 4
 * multiplicative (reading C23, RGAT's multiplicative logit q_i . k_j with one
 * query / key unit per head [ext]) ss * sd.  dl_dss / dl_dsd: its partial
 * derivatives (LeakyReLU'(0) = slope, C8). */
static double att_logit(int agg, double ss, double sd, double slope)
{
    return agg == 4 ? ss * sd : leaky(ss + sd, slope);
}
static double dlogit_dss(int agg, double ss, double sd, double slope)
{
    (void)ss;
    return agg == 4 ? sd : ((ss + sd) > 0 ? 1.0 : slope);
}
static double dlogit_dsd(int agg, double ss, double sd, double slope)
{
    (void)sd;
    return agg == 4 ? ss : ((ss + sd) > 0 ? 1.0 : slope);
}

/* GAT with the softmax ACROSS relations (reading
 * C5' in DESIGN.md; the PyG RGATConv default): for destination (t, i) and
 * head h, alpha_e = softmax over ALL in-edges of (t, i), whatever their
 * relation, of l_e = LeakyReLU(s_src[col_e] + s_dst[(r_e, i)]); each
 * relation's row still receives only its own edges' terms,
 * Z[(r,i)] = sum_{e in row (r,i)} alpha_e Y[col_e], so the semantic fusion
 * sum over r (O4) is the attention-weighted sum over all neighbours.
 * Edge order inside the union: relation ascending, then the row's order. */
static void gat_xrel_fwd(int T, int R, const int32_t *rel_src, const int32_t *rel_dst,
                         const int32_t *n_src, const int32_t *n_dst,
                         int64_t N, const int32_t *src, const int32_t *dst, const int64_t *eid,
                         const int32_t *edge_type, int64_t E,
                         const int32_t *rel_y_off, const int32_t *y_src,
                         int D, int H, double slope, const double *Y, const double *s_src,
                         const double *s_dst, const int64_t *rro, double *Z, double *deg_out,
                         double *alpha)
{
    int dh = D / H;
    int64_t **ptr = (int64_t **)malloc(sizeof(int64_t *) * R);
    int64_t **list = (int64_t **)malloc(sizeof(int64_t *) * R);
    for (int r = 0; r < R; r++)
        relation_rows(R, rel_src, rel_dst, n_src, n_dst, r, N, src, dst, eid, edge_type, E,
                      &ptr[r], &list[r]);
    for (int t = 0; t < T; t++)
        for (int32_t i = 0; i < n_dst[t]; i++) {
            for (int r = 0; r < R; r++)
                if (rel_dst[r] == t) deg_out[rro[r] + i] = (double)(ptr[r][i + 1] - ptr[r][i]);
            for (int h = 0; h < H; h++) {
                double m = -INFINITY, sum = 0.0;
                for (int r = 0; r < R; r++) {
                    if (rel_dst[r] != t) continue;
                    for (int64_t k = ptr[r][i]; k < ptr[r][i + 1]; k++) {
                        int32_t u = yrow_of(rel_y_off, y_src, r, src[list[r][k]]);
                        double l = leaky(s_src[(int64_t)u * H + h] + s_dst[(rro[r] + i) * H + h], slope);
                        if (l > m) m = l;
                    }
                }
                for (int r = 0; r < R; r++) {
                    if (rel_dst[r] != t) continue;
                    for (int64_t k = ptr[r][i]; k < ptr[r][i + 1]; k++) {
                        int32_t u = yrow_of(rel_y_off, y_src, r, src[list[r][k]]);
                        sum += exp(leaky(s_src[(int64_t)u * H + h] + s_dst[(rro[r] + i) * H + h], slope) - m);
                    }
                }
                for (int r = 0; r < R; r++) {
                    if (rel_dst[r] != t) continue;
                    double *z = Z + (rro[r] + i) * D;
                    for (int64_t k = ptr[r][i]; k < ptr[r][i + 1]; k++) {
                        int32_t u = yrow_of(rel_y_off, y_src, r, src[list[r][k]]);
                        double a = exp(leaky(s_src[(int64_t)u * H + h] + s_dst[(rro[r] + i) * H + h], slope) - m) / sum;
                        if (alpha) alpha[list[r][k] * H + h] = a;
                        for (int c = 0; c < dh; c++) z[h * dh + c] += a * Y[(int64_t)u * D + h * dh + c];
                    }
                }
            }
        }
    for (int r = 0; r < R; r++) { free(ptr[r]); free(list[r]); }
    free(ptr); free(list);
}

/* Adjoint of gat_xrel_fwd.  The fusion sum gives dZ[(r,i)] = G_t[i] for every
 * row of (t, i), so with o = sum_r Z[(r,i)] (head h):
 *   dalpha_e = <g_h, y_e>,  dl_e = alpha_e (dalpha_e - sum_{e' in union} alpha_e' dalpha_e'). */
static void gat_xrel_bwd(int T, int R, const int32_t *rel_src, const int32_t *rel_dst,
                         const int32_t *n_src, const int32_t *n_dst,
                         int64_t N, const int32_t *src, const int32_t *dst, const int64_t *eid,
                         const int32_t *edge_type, int64_t E,
                         const int32_t *rel_y_off, const int32_t *y_src,
                         int D, int H, double slope, const double *Gt, const double *Y,
                         const double *s_src, const double *s_dst, const int64_t *rro,
                         const int64_t *tdo, double *dY, double *ds_src, double *ds_dst)
{
    int dh = D / H;
    int64_t **ptr = (int64_t **)malloc(sizeof(int64_t *) * R);
    int64_t **list = (int64_t **)malloc(sizeof(int64_t *) * R);
    for (int r = 0; r < R; r++)
        relation_rows(R, rel_src, rel_dst, n_src, n_dst, r, N, src, dst, eid, edge_type, E,
                      &ptr[r], &list[r]);
    for (int t = 0; t < T; t++)
        for (int32_t i = 0; i < n_dst[t]; i++) {
            const double *g = Gt + (tdo[t] + i) * D;
            for (int h = 0; h < H; h++) {
                double m = -INFINITY, sum = 0.0, za = 0.0;
                for (int r = 0; r < R; r++) {
                    if (rel_dst[r] != t) continue;
                    for (int64_t k = ptr[r][i]; k < ptr[r][i + 1]; k++) {
                        int32_t u = yrow_of(rel_y_off, y_src, r, src[list[r][k]]);
                        double l = leaky(s_src[(int64_t)u * H + h] + s_dst[(rro[r] + i) * H + h], slope);
                        if (l > m) m = l;
                    }
                }
                for (int r = 0; r < R; r++) {
                    if (rel_dst[r] != t) continue;
                    for (int64_t k = ptr[r][i]; k < ptr[r][i + 1]; k++) {
                        int32_t u = yrow_of(rel_y_off, y_src, r, src[list[r][k]]);
                        sum += exp(leaky(s_src[(int64_t)u * H + h] + s_dst[(rro[r] + i) * H + h], slope) - m);
                    }
                }
                for (int r = 0; r < R; r++) {
                    if (rel_dst[r] != t) continue;
                    for (int64_t k = ptr[r][i]; k < ptr[r][i + 1]; k++) {
                        int32_t u = yrow_of(rel_y_off, y_src, r, src[list[r][k]]);
                        double a = exp(leaky(s_src[(int64_t)u * H + h] + s_dst[(rro[r] + i) * H + h], slope) - m) / sum;
                        double da = 0.0;
                        for (int c = 0; c < dh; c++) da += g[h * dh + c] * Y[(int64_t)u * D + h * dh + c];
                        za += a * da;
                    }
                }
                for (int r = 0; r < R; r++) {
                    if (rel_dst[r] != t) continue;
                    int64_t row = rro[r] + i;
                    for (int64_t k = ptr[r][i]; k < ptr[r][i + 1]; k++) {
                        int32_t u = yrow_of(rel_y_off, y_src, r, src[list[r][k]]);
                        double pre = s_src[(int64_t)u * H + h] + s_dst[row * H + h];
                        double a = exp(leaky(pre, slope) - m) / sum;
                        double da = 0.0;
                        for (int c = 0; c < dh; c++) {
                            da += g[h * dh + c] * Y[(int64_t)u * D + h * dh + c];
                            dY[(int64_t)u * D + h * dh + c] += a * g[h * dh + c];
                        }
                        double dpre = a * (da - za) * (pre > 0 ? 1.0 : slope);
                        ds_src[(int64_t)u * H + h] += dpre;
                        ds_dst[row * H + h] += dpre;
                    }
                }
            }
        }
    for (int r = 0; r < R; r++) { free(ptr[r]); free(list[r]); }
    free(ptr); free(list);
}

void oracle_aggregate_fwd(int T, int R, const int32_t *rel_src, const int32_t *rel_dst,
                          const int32_t *n_src, const int32_t *n_dst,
                          int64_t N, const int32_t *src, const int32_t *dst, const int64_t *eid,
                          const int32_t *edge_type, int64_t E,
                          const int32_t *rel_y_off, const int32_t *y_src,
                          int agg, int D, int H, double slope,
                          const double *Y, const double *s_src, const double *s_dst,
                          double *Z, double *deg_out, double *alpha)
{
    (void)T;
    int64_t rows = 0;
    int64_t *rro = (int64_t *)malloc(sizeof(int64_t) * (R + 1));
    for (int r = 0; r < R; r++) { rro[r] = rows; rows += n_dst[rel_dst[r]]; }
    rro[R] = rows;
    memset(Z, 0, sizeof(double) * rows * D);
    memset(deg_out, 0, sizeof(double) * rows);
    int dh = D / H;
    if (agg == 3) {
        gat_xrel_fwd(T, R, rel_src, rel_dst, n_src, n_dst, N, src, dst, eid, edge_type, E,
                     rel_y_off, y_src, D, H, slope, Y, s_src, s_dst, rro, Z, deg_out, alpha);
        free(rro);
        return;
    }
    for (int r = 0; r < R; r++) {
        /* lines 254-256: IndexSelect of the relation's sources, DstIndex kept */
        int64_t *ptr, *list;
        relation_rows(R, rel_src, rel_dst, n_src, n_dst, r, N, src, dst, eid, edge_type, E, &ptr, &list);
        for (int32_t i = 0; i < n_dst[rel_dst[r]]; i++) {
            int64_t row = rro[r] + i;
            double deg = (double)(ptr[i + 1] - ptr[i]);
            deg_out[row] = deg;
            double *z = Z + row * D;
            if (agg != 2 && agg != 4) {
                /* line 260: Aggregate = segment sum (mean: / |segment|, C1) */
                for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
                    const double *y = Y + (int64_t)yrow_of(rel_y_off, y_src, r, src[list[k]]) * D;
                    for (int d = 0; d < D; d++) z[d] += y[d];
                }
                if (agg == 1 && deg > 0)
                    for (int d = 0; d < D; d++) z[d] /= deg;
                continue;
            }
            /* GAT (C5, C6, C8; agg 4: multiplicative logit, C23): per head,
             * softmax over the segment of l_e = LeakyReLU(s_src[col_e] +
             * s_dst[row]) (agg 4: s_src[col_e] s_dst[row]), then sum alpha_e Y[col_e] */
            for (int h = 0; h < H; h++) {
                double m = -INFINITY, sum = 0.0;
                for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
                    int32_t u = yrow_of(rel_y_off, y_src, r, src[list[k]]);
                    double l = att_logit(agg, s_src[(int64_t)u * H + h], s_dst[row * H + h], slope);
                    if (l > m) m = l;
                }
                for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
                    int32_t u = yrow_of(rel_y_off, y_src, r, src[list[k]]);
                    sum += exp(att_logit(agg, s_src[(int64_t)u * H + h], s_dst[row * H + h], slope) - m);
                }
                for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
                    int32_t u = yrow_of(rel_y_off, y_src, r, src[list[k]]);
                    double a = exp(att_logit(agg, s_src[(int64_t)u * H + h], s_dst[row * H + h], slope) - m) / sum;
                    if (alpha) alpha[list[k] * H + h] = a;
                    for (int c = 0; c < dh; c++) z[h * dh + c] += a * Y[(int64_t)u * D + h * dh + c];
                }
            }
        }
        free(ptr); free(list);
    }
    free(rro);
}

/* ------------------------------------------------------------------------ */
/* O4. Semantic fusion ("combining the results from the previous     */
/* stage"), reading C2/C4/C10: H_t[i] = act(R0_t[i] + b_t + sum_{r:t(r)=t}   */
/* Z[(r,i)]); act: 0 none, 1 ReLU.                                           */
/* ------------------------------------------------------------------------ */
void oracle_fuse(int T, int R, const int32_t *rel_dst, const int32_t *n_dst, int D, int act,
                 const double *Z, const double *R0, const double *bias, const double *beta,
                 double *Hout)
{
    int64_t *tdo = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    tdo[0] = 0;
    for (int t = 0; t < T; t++) tdo[t + 1] = tdo[t] + n_dst[t];
    for (int t = 0; t < T; t++)
        for (int32_t i = 0; i < n_dst[t]; i++)
            for (int d = 0; d < D; d++) {
                double v = 0.0;
                if (R0) v += R0[(tdo[t] + i) * D + d];
                if (bias) v += bias[(int64_t)t * D + d];
                int64_t row = 0;
                for (int r = 0; r < R; r++) {
                    /* beta: HAN semantic-attention weights (O4'), NULL: 1 */
                    if (rel_dst[r] == t) v += (beta ? beta[r] : 1.0) * Z[(row + i) * D + d];
                    row += n_dst[rel_dst[r]];
                }
                if (act == 1 && v < 0) v = 0;
                Hout[(tdo[t] + i) * D + d] = v;
            }
    free(tdo);
}

/* ------------------------------------------------------------------------ */
/* O4'. HAN semantic-attention fusion (P:L123 leaves */
/* the fusion rule open: "combining the results"; reading C22, HAN's          */
/* semantic-level attention [ext]).  Per relation r into type t:              */
/*   w_r    = (1/n_t) sum_{i<n_t} q . tanh(Ws^T Z[(r,i)] + bs)                */
/*   beta_r = exp(w_r) / sum_{r': t(r')=t} exp(w_r')                          */
/* and O4 fuses with weights: H_t[i] = act(R0 + b + sum_r beta_r Z[(r,i)]).   */
/* Ws [D,A], bs [A], q [A].  A type without destinations gets w = 0.          */
/* ------------------------------------------------------------------------ */
void oracle_sem_att(int T, int R, const int32_t *rel_dst, const int32_t *n_dst, int D, int A,
                    const double *Z, const double *Ws, const double *bs, const double *q,
                    double *w, double *beta)
{
    double *a = (double *)malloc(sizeof(double) * A);
    int64_t row = 0;
    for (int r = 0; r < R; r++) {
        int32_t nt = n_dst[rel_dst[r]];
        double acc = 0.0;
        for (int32_t i = 0; i < nt; i++, row++) {
            const double *z = Z + row * D;
            for (int c = 0; c < A; c++) {
                double v = bs[c];
                for (int d = 0; d < D; d++) v += z[d] * Ws[(int64_t)d * A + c];
                a[c] = v;
            }
            double s = 0.0;
            for (int c = 0; c < A; c++) s += q[c] * tanh(a[c]);
            acc += s;
        }
        w[r] = nt > 0 ? acc / nt : 0.0;
    }
    for (int t = 0; t < T; t++) {
        double m = -INFINITY, sum = 0.0;
        for (int r = 0; r < R; r++) if (rel_dst[r] == t && w[r] > m) m = w[r];
        for (int r = 0; r < R; r++) if (rel_dst[r] == t) sum += exp(w[r] - m);
        for (int r = 0; r < R; r++) if (rel_dst[r] == t) beta[r] = exp(w[r] - m) / sum;
    }
    free(a);
}

/* O5a'. Adjoint of O4' + the weighted sum of O4, given G = dL/d(pre-       */
/* activation fused value) (type-major, from O5a):                           */
/*   dbeta_r = sum_i <G_t[i], Z[(r,i)]>                                       */
/*   dw_r    = beta_r (dbeta_r - sum_{r': t(r')=t} beta_r' dbeta_r')          */
/*   g_a     = (dw_r / n_t) q (.) (1 - tanh^2(a)),  a = Ws^T Z[(r,i)] + bs    */
/*   dZ[(r,i)] = beta_r G_t[i] + Ws g_a                                       */
/*   dWs += Z[(r,i)] (x) g_a;  dbs += g_a;  dq += (dw_r / n_t) tanh(a)         */
void oracle_sem_att_bwd(int T, int R, const int32_t *rel_dst, const int32_t *n_dst, int D, int A,
                        const double *Z, const double *Ws, const double *bs, const double *q,
                        const double *beta, const double *G,
                        double *dZ, double *dWs, double *dbs, double *dq)
{
    int64_t *tdo = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    tdo[0] = 0;
    for (int t = 0; t < T; t++) tdo[t + 1] = tdo[t] + n_dst[t];
    double *dbeta = (double *)calloc(R, sizeof(double));
    double *dw = (double *)calloc(R, sizeof(double));
    double *a = (double *)malloc(sizeof(double) * A);
    double *ga = (double *)malloc(sizeof(double) * A);
    memset(dWs, 0, sizeof(double) * D * A);
    memset(dbs, 0, sizeof(double) * A);
    memset(dq, 0, sizeof(double) * A);
    int64_t row = 0;
    for (int r = 0; r < R; r++) {
        int t = rel_dst[r];
        for (int32_t i = 0; i < n_dst[t]; i++, row++)
            for (int d = 0; d < D; d++) dbeta[r] += G[(tdo[t] + i) * D + d] * Z[row * D + d];
    }
    for (int r = 0; r < R; r++) {
        double s = 0.0;
        for (int r2 = 0; r2 < R; r2++) if (rel_dst[r2] == rel_dst[r]) s += beta[r2] * dbeta[r2];
        dw[r] = beta[r] * (dbeta[r] - s);
    }
    row = 0;
    for (int r = 0; r < R; r++) {
        int t = rel_dst[r];
        int32_t nt = n_dst[t];
        for (int32_t i = 0; i < nt; i++, row++) {
            const double *z = Z + row * D;
            for (int c = 0; c < A; c++) {
                double v = bs[c];
                for (int d = 0; d < D; d++) v += z[d] * Ws[(int64_t)d * A + c];
                a[c] = v;
            }
            for (int c = 0; c < A; c++) {
                double th = tanh(a[c]);
                ga[c] = dw[r] / nt * q[c] * (1.0 - th * th);
                dbs[c] += ga[c];
                dq[c] += dw[r] / nt * th;
            }
            for (int d = 0; d < D; d++) {
                double v = beta[r] * G[(tdo[t] + i) * D + d];
                for (int c = 0; c < A; c++) {
                    v += Ws[(int64_t)d * A + c] * ga[c];
                    dWs[(int64_t)d * A + c] += z[d] * ga[c];
                }
                dZ[row * D + d] = v;
            }
        }
    }
    free(dbeta); free(dw); free(a); free(ga); free(tdo);
}

/* O5a. Fusion backward: G = dH * act'(H) (ReLU' = 1[H > 0]), which is also   */
/* dZ of every relation into the type and dR0; dbias_t = sum_i G_t[i].       */
void oracle_fuse_bwd(int T, const int32_t *n_dst, int D, int act,
                     const double *dH, const double *Hv, double *G, double *dbias)
{
    int64_t row = 0;
    for (int t = 0; t < T; t++) {
        for (int d = 0; d < D; d++) dbias[(int64_t)t * D + d] = 0.0;
        for (int32_t i = 0; i < n_dst[t]; i++, row++)
            for (int d = 0; d < D; d++) {
                double g = dH[row * D + d];
                if (act == 1 && !(Hv[row * D + d] > 0)) g = 0.0;
                G[row * D + d] = g;
                dbias[(int64_t)t * D + d] += g;
            }
    }
}

/* ------------------------------------------------------------------------ */
/* O5b. Aggregation backward ("backward pass on GPU for gradient      */
/* computation"), the adjoint of O3, relation by relation.  G is the type-   */
/* major gradient of the fused output; dZ[(r,i)] = G_{t(r)}[i].  Outputs     */
/* dY (aggregation term only), ds_src [U,H], ds_dst [rows,H] (GAT).          */
/* ------------------------------------------------------------------------ */
void oracle_aggregate_bwd(int T, int R, const int32_t *rel_src, const int32_t *rel_dst,
                          const int32_t *n_src, const int32_t *n_dst,
                          int64_t N, const int32_t *src, const int32_t *dst, const int64_t *eid,
                          const int32_t *edge_type, int64_t E,
                          const int32_t *rel_y_off, const int32_t *y_src, int64_t U,
                          int agg, int D, int H, double slope, int g_rows,
                          const double *Gt, const double *Y, const double *s_src, const double *s_dst,
                          double *dY, double *ds_src, double *ds_dst)
{
    int64_t *tdo = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    tdo[0] = 0;
    for (int t = 0; t < T; t++) tdo[t + 1] = tdo[t] + n_dst[t];
    int64_t rows = 0;
    int64_t *rro = (int64_t *)malloc(sizeof(int64_t) * (R + 1));
    for (int r = 0; r < R; r++) { rro[r] = rows; rows += n_dst[rel_dst[r]]; }
    rro[R] = rows;
    memset(dY, 0, sizeof(double) * U * D);
    if (agg >= 2) { memset(ds_src, 0, sizeof(double) * U * H); memset(ds_dst, 0, sizeof(double) * rows * H); }
    if (g_rows && agg == 3) { free(rro); free(tdo); abort(); }   /* not defined for xrel */
    int dh = D / H;
    if (agg == 3) {
        gat_xrel_bwd(T, R, rel_src, rel_dst, n_src, n_dst, N, src, dst, eid, edge_type, E,
                     rel_y_off, y_src, D, H, slope, Gt, Y, s_src, s_dst, rro, tdo, dY, ds_src,
                     ds_dst);
        free(rro); free(tdo);
        return;
    }
    for (int r = 0; r < R; r++) {
        int t = rel_dst[r];
        int64_t *ptr, *list;
        relation_rows(R, rel_src, rel_dst, n_src, n_dst, r, N, src, dst, eid, edge_type, E, &ptr, &list);
        for (int32_t i = 0; i < n_dst[t]; i++) {
            int64_t row = rro[r] + i;
            /* dZ[(r,i)] = G_t[i] (plain fusion), or a per-row gradient
             * (g_rows: HAN semantic attention, O4') */
            const double *g = g_rows ? Gt + row * D : Gt + (tdo[t] + i) * D;
            double deg = (double)(ptr[i + 1] - ptr[i]);
            if (agg != 2 && agg != 4) {
                double w = agg == 1 ? 1.0 / deg : 1.0;
                for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
                    int32_t u = yrow_of(rel_y_off, y_src, r, src[list[k]]);
                    for (int d = 0; d < D; d++) dY[(int64_t)u * D + d] += w * g[d];
                }
                continue;
            }
            for (int h = 0; h < H; h++) {
                /* recompute alpha of the segment (forward O3) */
                double m = -INFINITY, sum = 0.0, za = 0.0;
                for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
                    int32_t u = yrow_of(rel_y_off, y_src, r, src[list[k]]);
                    double l = att_logit(agg, s_src[(int64_t)u * H + h], s_dst[row * H + h], slope);
                    if (l > m) m = l;
                }
                for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
                    int32_t u = yrow_of(rel_y_off, y_src, r, src[list[k]]);
                    sum += exp(att_logit(agg, s_src[(int64_t)u * H + h], s_dst[row * H + h], slope) - m);
                }
                /* z_h = sum_e alpha_e y_e  =>  dalpha_e = <g_h, y_e>;
                 * softmax: dl_e = alpha_e (dalpha_e - sum_e' alpha_e' dalpha_e') */
                for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
                    int32_t u = yrow_of(rel_y_off, y_src, r, src[list[k]]);
                    double a = exp(att_logit(agg, s_src[(int64_t)u * H + h], s_dst[row * H + h], slope) - m) / sum;
                    double da = 0.0;
                    for (int c = 0; c < dh; c++) da += g[h * dh + c] * Y[(int64_t)u * D + h * dh + c];
                    za += a * da;
                }
                for (int64_t k = ptr[i]; k < ptr[i + 1]; k++) {
                    int32_t u = yrow_of(rel_y_off, y_src, r, src[list[k]]);
                    double ss = s_src[(int64_t)u * H + h], sd = s_dst[row * H + h];
                    double a = exp(att_logit(agg, ss, sd, slope) - m) / sum;
                    double da = 0.0;
                    for (int c = 0; c < dh; c++) {
                        da += g[h * dh + c] * Y[(int64_t)u * D + h * dh + c];
                        dY[(int64_t)u * D + h * dh + c] += a * g[h * dh + c];
                    }
                    double dl = a * (da - za);
                    ds_src[(int64_t)u * H + h] += dl * dlogit_dss(agg, ss, sd, slope);
                    ds_dst[row * H + h] += dl * dlogit_dsd(agg, ss, sd, slope);
                }
            }
        }
        free(ptr); free(list);
    }
    free(rro); free(tdo);
}

/* ------------------------------------------------------------------------ */
/* O5c. Projection backward: adjoint of O2.                                  */
/* dW_r = sum_u x_u^T dYtot_u, dYtot = dY + ds_src (x) a_src (score chain);  */
/* dW_root,t = sum_i X_t[i]^T G_t[i]; dX += dYtot W_r^T + G W_root^T;        */
/* s_dst chain: v_{r,h} = W_r[:,head h] a_dst^{r,h}; dX_t[i] += ds_dst v;    */
/* dW_r[:,head h] += (sum_i ds_dst X_t[i]) a_dst^T; da_dst, da_src.          */
/* dX may be NULL (layer 0).                                                 */
/* ------------------------------------------------------------------------ */
void oracle_project_bwd(int T, int R, const int32_t *rel_src, const int32_t *rel_dst,
                        const int32_t *n_src, const int32_t *n_dst,
                        int K, int D, int H,
                        const double *X, const int32_t *gather_ids,
                        const int32_t *rel_y_off, const int32_t *y_src,
                        const double *W_rel, const double *W_root, const double *att,
                        const double *Y, const double *dY, const double *G,
                        const double *ds_src, const double *ds_dst,
                        double *dX, int64_t x_rows, double *dW_rel, double *dW_root, double *datt)
{
    int64_t *tso = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    int64_t *tdo = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    tso[0] = tdo[0] = 0;
    for (int t = 0; t < T; t++) { tso[t + 1] = tso[t] + n_src[t]; tdo[t + 1] = tdo[t] + n_dst[t]; }
    int dh = D / H;
    memset(dW_rel, 0, sizeof(double) * R * K * D);
    if (dW_root) memset(dW_root, 0, sizeof(double) * T * K * D);
    if (datt) memset(datt, 0, sizeof(double) * R * 2 * D);
    if (dX) memset(dX, 0, sizeof(double) * x_rows * K);
    for (int r = 0; r < R; r++) {
        const double *W = W_rel + (int64_t)r * K * D;
        double *dW = dW_rel + (int64_t)r * K * D;
        const double *a_src = att ? att + (int64_t)r * 2 * D : NULL;
        int32_t u0 = rel_y_off[r], nu = rel_y_off[r + 1] - rel_y_off[r];
        /* dYt[u] = dY[u] + ds_src[u,h] a_src^{r,h} (the s_src term of O2) */
        double *dyt = (double *)malloc(sizeof(double) * D * (nu > 0 ? nu : 1));
        for (int32_t q = 0; q < nu; q++) {
            int32_t u = u0 + q;
            for (int d = 0; d < D; d++) dyt[(int64_t)q * D + d] = dY[(int64_t)u * D + d];
            if (att)
                for (int h = 0; h < H; h++)
                    for (int c = 0; c < dh; c++) {
                        dyt[(int64_t)q * D + h * dh + c] += ds_src[(int64_t)u * H + h] * a_src[h * dh + c];
                        datt[(int64_t)r * 2 * D + h * dh + c] += ds_src[(int64_t)u * H + h] * Y[(int64_t)u * D + h * dh + c];
                    }
        }
        /* dW_r[k,:] = sum_u X[src u, k] dYt[u]  (u ascending, row k per thread) */
        #pragma omp parallel for schedule(static)
        for (int k = 0; k < K; k++)
            for (int32_t q = 0; q < nu; q++) {
                int64_t xr = tso[rel_src[r]] + y_src[u0 + q];
                if (gather_ids) xr = gather_ids[xr];
                double xk = X[xr * K + k];
                for (int d = 0; d < D; d++) dW[(int64_t)k * D + d] += xk * dyt[(int64_t)q * D + d];
            }
        /* dX[src u] += dYt[u] W_r^T  (distinct sources within relation r) */
        if (dX) {
            #pragma omp parallel for schedule(static)
            for (int32_t q = 0; q < nu; q++) {
                int64_t xr = tso[rel_src[r]] + y_src[u0 + q];
                if (gather_ids) xr = gather_ids[xr];
                for (int k = 0; k < K; k++) {
                    double acc = 0.0;
                    for (int d = 0; d < D; d++) acc += dyt[(int64_t)q * D + d] * W[(int64_t)k * D + d];
                    dX[xr * K + k] += acc;
                }
            }
        }
        free(dyt);
    }
    if (W_root) {
        for (int t = 0; t < T; t++) {
            const double *W = W_root + (int64_t)t * K * D;
            double *dW = dW_root + (int64_t)t * K * D;
            /* dW_root,t[k,:] = sum_i X_t[i, k] G_t[i] */
            #pragma omp parallel for schedule(static)
            for (int k = 0; k < K; k++)
                for (int32_t i = 0; i < n_dst[t]; i++) {
                    int64_t xr = tso[t] + i;
                    if (gather_ids) xr = gather_ids[xr];
                    const double *g = G + (tdo[t] + i) * D;
                    double xk = X[xr * K + k];
                    for (int d = 0; d < D; d++) dW[(int64_t)k * D + d] += xk * g[d];
                }
            if (dX) {
                #pragma omp parallel for schedule(static)
                for (int32_t i = 0; i < n_dst[t]; i++) {
                    int64_t xr = tso[t] + i;
                    if (gather_ids) xr = gather_ids[xr];
                    const double *g = G + (tdo[t] + i) * D;
                    for (int k = 0; k < K; k++) {
                        double acc = 0.0;
                        for (int d = 0; d < D; d++) acc += g[d] * W[(int64_t)k * D + d];
                        dX[xr * K + k] += acc;
                    }
                }
            }
        }
    }
    if (att) {
        int64_t row0 = 0;
        for (int r = 0; r < R; r++) {
            const double *W = W_rel + (int64_t)r * K * D;
            double *dW = dW_rel + (int64_t)r * K * D;
            const double *a_dst = att + (int64_t)r * 2 * D + D;
            int t = rel_dst[r];
            int32_t nt = n_dst[t];
            /* s_dst = sum_c (x W_r)[hc] a_dst[hc]  =>  d/d(xW)[hc] = ds_dst[h] a_dst[hc];
             * gd[i, d] = ds_dst[(r,i), h(d)] a_dst[d] */
            double *gd = (double *)malloc(sizeof(double) * D * (nt > 0 ? nt : 1));
            for (int32_t i = 0; i < nt; i++)
                for (int h = 0; h < H; h++)
                    for (int c = 0; c < dh; c++)
                        gd[(int64_t)i * D + h * dh + c] = ds_dst[(row0 + i) * H + h] * a_dst[h * dh + c];
            /* datt_dst[d] += ds_dst[h(d)] (x W_r)[d], i ascending */
            double *hv = (double *)malloc(sizeof(double) * D);
            for (int32_t i = 0; i < nt; i++) {
                int64_t xr = tso[t] + i;
                if (gather_ids) xr = gather_ids[xr];
                const double *x = X + xr * K;
                for (int d = 0; d < D; d++) hv[d] = 0.0;
                for (int k = 0; k < K; k++)
                    for (int d = 0; d < D; d++) hv[d] += x[k] * W[(int64_t)k * D + d];
                for (int h = 0; h < H; h++)
                    for (int c = 0; c < dh; c++)
                        datt[(int64_t)r * 2 * D + D + h * dh + c] += ds_dst[(row0 + i) * H + h] * hv[h * dh + c];
            }
            free(hv);
            /* dW_r[k, d] += x_i[k] gd[i, d], i ascending */
            #pragma omp parallel for schedule(static)
            for (int k = 0; k < K; k++)
                for (int32_t i = 0; i < nt; i++) {
                    int64_t xr = tso[t] + i;
                    if (gather_ids) xr = gather_ids[xr];
                    double xk = X[xr * K + k];
                    for (int d = 0; d < D; d++) dW[(int64_t)k * D + d] += xk * gd[(int64_t)i * D + d];
                }
            if (dX) {
                #pragma omp parallel for schedule(static)
                for (int32_t i = 0; i < nt; i++) {
                    int64_t xr = tso[t] + i;
                    if (gather_ids) xr = gather_ids[xr];
                    for (int k = 0; k < K; k++)
                        for (int d = 0; d < D; d++)
                            dX[xr * K + k] += gd[(int64_t)i * D + d] * W[(int64_t)k * D + d];
                }
            }
            free(gd);
            row0 += nt;
        }
    }
    free(tso); free(tdo);
}

/* ------------------------------------------------------------------------ */
/* O6. Aggregate-first RGCN input layer (DESIGN.md  */
/* §9).  Alg. 1 applied to the RAW features, relation by        */
/* relation: Xagg[(r,i)] = sum (mean: / |segment|) over the segment of       */
/* X_s(r)[src e]; then the projection of P:L119 on the aggregated rows,      */
/* Z[(r,i)] = Xagg[(r,i)] W_r, and the root term R0_t = X_t W_root,t.  By    */
/* linearity Z equals O3(O2(X)) -- tests/test_oracle_aggfirst.py pins that.  */
/* ------------------------------------------------------------------------ */
void oracle_aggregate_features(int T, int R, const int32_t *rel_src, const int32_t *rel_dst,
                               const int32_t *n_src, const int32_t *n_dst,
                               int64_t N, const int32_t *src, const int32_t *dst,
                               const int64_t *eid, const int32_t *edge_type, int64_t E,
                               int agg, int K, const double *X, const int32_t *gather_ids,
                               double *Xagg)
{
    int64_t *tso = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    tso[0] = 0;
    for (int t = 0; t < T; t++) tso[t + 1] = tso[t] + n_src[t];
    int64_t row0 = 0;
    for (int r = 0; r < R; r++) {
        int64_t *ptr, *list;
        relation_rows(R, rel_src, rel_dst, n_src, n_dst, r, N, src, dst, eid, edge_type, E, &ptr, &list);
        for (int32_t i = 0; i < n_dst[rel_dst[r]]; i++) {
            double *z = Xagg + (row0 + i) * K;
            for (int k = 0; k < K; k++) z[k] = 0.0;
            for (int64_t q = ptr[i]; q < ptr[i + 1]; q++) {
                const double *x = xrow(X, K, gather_ids, tso, rel_src[r], src[list[q]]);
                for (int k = 0; k < K; k++) z[k] += x[k];
            }
            double deg = (double)(ptr[i + 1] - ptr[i]);
            if (agg == 1 && deg > 0)
                for (int k = 0; k < K; k++) z[k] /= deg;
        }
        row0 += n_dst[rel_dst[r]];
        free(ptr); free(list);
    }
    free(tso);
}

void oracle_project_aggregated(int T, int R, const int32_t *rel_dst, const int32_t *n_src,
                               const int32_t *n_dst, int K, int D, const double *Xagg,
                               const double *X, const int32_t *gather_ids,
                               const double *W_rel, const double *W_root, double *Z, double *R0)
{
    int64_t *tso = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    tso[0] = 0;
    for (int t = 0; t < T; t++) tso[t + 1] = tso[t] + n_src[t];
    int64_t row0 = 0;
    for (int r = 0; r < R; r++) {
        const double *W = W_rel + (int64_t)r * K * D;
        for (int32_t i = 0; i < n_dst[rel_dst[r]]; i++) {
            const double *x = Xagg + (row0 + i) * K;
            double *z = Z + (row0 + i) * D;
            for (int d = 0; d < D; d++) {
                double s = 0.0;
                for (int k = 0; k < K; k++) s += x[k] * W[(int64_t)k * D + d];
                z[d] = s;
            }
        }
        row0 += n_dst[rel_dst[r]];
    }
    if (W_root) {
        int64_t o = 0;
        for (int t = 0; t < T; t++) {
            const double *W = W_root + (int64_t)t * K * D;
            for (int32_t i = 0; i < n_dst[t]; i++) {
                const double *x = xrow(X, K, gather_ids, tso, t, i);
                for (int d = 0; d < D; d++) {
                    double s = 0.0;
                    for (int k = 0; k < K; k++) s += x[k] * W[(int64_t)k * D + d];
                    R0[(o + i) * D + d] = s;
                }
            }
            o += n_dst[t];
        }
    }
    free(tso);
}

/* Adjoint: dW_r = sum_i Xagg[(r,i)]^T G_t(r)[i] (every Z row (r,i) feeds
 * H_t(r)[i] through the fusion sum), dW_root,t = sum_i X_t[i]^T G_t[i]. */
void oracle_project_aggregated_bwd(int T, int R, const int32_t *rel_dst, const int32_t *n_src,
                                   const int32_t *n_dst, int K, int D, const double *Xagg,
                                   const double *X, const int32_t *gather_ids, const double *G,
                                   double *dW_rel, double *dW_root)
{
    int64_t *tso = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    int64_t *tdo = (int64_t *)malloc(sizeof(int64_t) * (T + 1));
    tso[0] = tdo[0] = 0;
    for (int t = 0; t < T; t++) { tso[t + 1] = tso[t] + n_src[t]; tdo[t + 1] = tdo[t] + n_dst[t]; }
    memset(dW_rel, 0, sizeof(double) * R * K * D);
    int64_t row0 = 0;
    for (int r = 0; r < R; r++) {
        double *W = dW_rel + (int64_t)r * K * D;
        int t = rel_dst[r];
        for (int32_t i = 0; i < n_dst[t]; i++) {
            const double *x = Xagg + (row0 + i) * K;
            const double *g = G + (tdo[t] + i) * D;
            for (int k = 0; k < K; k++)
                for (int d = 0; d < D; d++) W[(int64_t)k * D + d] += x[k] * g[d];
        }
        row0 += n_dst[t];
    }
    if (dW_root) {
        memset(dW_root, 0, sizeof(double) * T * K * D);
        for (int t = 0; t < T; t++) {
            double *W = dW_root + (int64_t)t * K * D;
            for (int32_t i = 0; i < n_dst[t]; i++) {
                const double *x = xrow(X, K, gather_ids, tso, t, i);
                const double *g = G + (tdo[t] + i) * D;
                for (int k = 0; k < K; k++)
                    for (int d = 0; d < D; d++) W[(int64_t)k * D + d] += x[k] * g[d];
            }
        }
    }
    free(tso); free(tdo);
}

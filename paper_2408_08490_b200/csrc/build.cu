// build.cu -- A1: semantic graph build (Alg. 2) as a
// merged segmented CSR + CSC, on the GPU, with a kernel count independent of
// the number of relations R.
//
// Alg. 2 runs, per layer, 1 gather (line 316) + R compares (318) + R
// index-selects (319): 2R+1 short kernels that the paper offloads to the CPU
// (lines 299-336).  Here the relation of each edge only decides a KEY,
//   key(e) = rel_row_off[r(e)] + dst(e)      (merged row, relation-major),
// and one counting sort by key performs every relation's selection at once:
//   k_classify   EdgeTypeLayer gather + validation + row histogram + source
//                presence flags per (relation, source) slot
//   scan         row_ptr and the compact Y-row numbering (one scan over both)
//   k_finish     rel_y_off, y_src, slot_y, U
//   k_scatter    unstable atomic placement into rows + column histogram
//   scan         col_ptr
//   k_fix_rows   warp per row: sort by original column (restores Alg. 2's
//                column order, so the result is bit-exact and deterministic),
//                then CSC placement
//   k_fix_cols   thread per Y row: sort CSC entries by CSR position
//   k_sort_long  the same two sorts for segments longer than 32 (rank sort)
#include <cstdlib>
#include <vector>
#include "common.cuh"

namespace hf {


__global__ void k_classify(LayerMeta m, const int* __restrict__ src, const int* __restrict__ dst,
                           const long long* __restrict__ eid, const int* __restrict__ edge_type,
                           const long long* __restrict__ rel_off, long long E,
                           int* __restrict__ key_e, int* __restrict__ slot_e,
                           int* __restrict__ cnt, int* __restrict__ status) {
  __shared__ long long s_off[HF_MAX_R + 1];
  if (rel_off) {
    for (int i = threadIdx.x; i <= m.R; i += blockDim.x) s_off[i] = rel_off[i];
    __syncthreads();
  }
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.N) return;
  long long id = eid[e];
  int bad = 0, r = -1;
  int s = src[e], d = dst[e];
  if (id < 0 || id >= E) {
    bad = HIFUSE_ST_BAD_EDGE_ID;
  } else {
    // Alg. 2: EdgeTypeLayer = EdgeType[EdgeID] -- a gather, or for a
    // relation-major table the relation whose id range holds `id`
    if (rel_off) {
      int lo = 0, hi = m.R;                              // s_off[lo] <= id < s_off[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_off[mid] <= id) lo = mid; else hi = mid;
      }
      r = lo;
    } else {
      r = edge_type[id];
    }
    if (r < 0 || r >= m.R) bad = HIFUSE_ST_BAD_REL;
    else if (s < 0 || s >= m.n_src[m.rel_src[r]]) bad = HIFUSE_ST_BAD_SRC;
    else if (d < 0 || d >= m.n_dst[m.rel_dst[r]]) bad = HIFUSE_ST_BAD_DST;
  }
  if (bad) {
    atomicOr(status, bad);
    key_e[e] = -1;
    return;
  }
  int key = m.rel_row_off[r] + d;                        // lines 318-319, all r at once
  int slot = m.slot_off[r] + s;
  key_e[e] = key;
  slot_e[e] = slot;
  atomicAdd(&cnt[key], 1);
  cnt[m.rows + slot] = 1;                                // presence flag (idempotent)
}

// d_rel_edge_off[r] = lower bound of r in the (sorted) edge-type table.
__global__ void k_et_offsets(const int* __restrict__ et, long long E, int R,
                             long long* __restrict__ off) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > R) return;
  long long lo = 0, hi = E;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (et[mid] < r) lo = mid + 1; else hi = mid;
  }
  off[r] = r == R ? E : lo;
}

__global__ void k_et_check(const int* __restrict__ et, long long E, int R, int* __restrict__ status) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E) return;
  const int v = et[i];
  if (v < 0 || v >= R || (i > 0 && et[i - 1] > v)) atomicOr(status, HIFUSE_ST_UNSORTED_TYPES);
}

// pre = exclusive scan of [row counts | slot flags]; pre[rows] = valid edges,
// pre[rows + S] - pre[rows] = U.
__global__ void k_finish(LayerMeta m, const int* __restrict__ cnt, const int* __restrict__ pre,
                         int* __restrict__ row_ptr, int* __restrict__ rel_row_off,
                         int* __restrict__ rel_y_off, int* __restrict__ y_src,
                         int* __restrict__ slot_y, int* __restrict__ U_dev) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int nvalid = pre[m.rows];
  if (i <= m.rows) row_ptr[i] = pre[i];
  if (i < m.S) {
    int u = -1;
    if (cnt[m.rows + i]) {
      u = pre[m.rows + i] - nvalid;
      int r = upper_bound_i(m.slot_off, m.R + 1, i) - 1;
      y_src[u] = i - m.slot_off[r];
    }
    slot_y[i] = u;
  }
  if (i <= m.R) {
    rel_row_off[i] = m.rel_row_off[i];
    rel_y_off[i] = pre[m.rows + m.slot_off[i]] - nvalid;
  }
  if (i == 0) U_dev[0] = pre[m.rows + m.S] - nvalid;
}

__global__ void k_scatter(LayerMeta m, const int* __restrict__ key_e, const int* __restrict__ slot_e,
                          const int* __restrict__ row_ptr, const int* __restrict__ slot_y,
                          int* __restrict__ cur, int* __restrict__ ccnt, int* __restrict__ eperm,
                          int* __restrict__ col, int* __restrict__ csc_pos,
                          int* __restrict__ csc_row) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.N) return;
  int nvalid = row_ptr[m.rows];
  if (e >= nvalid) {  // tail positions [nvalid, N): exactly one writer each
    eperm[e] = -1; col[e] = -1;
    if (csc_pos) { csc_pos[e] = -1; csc_row[e] = -1; }
  }
  int key = key_e[e];
  if (key < 0) return;
  int pos = row_ptr[key] + atomicAdd(&cur[key], 1);
  int c = slot_y[slot_e[e]];
  eperm[pos] = e;
  col[pos] = c;
  if (csc_pos) atomicAdd(&ccnt[c], 1);
}

// Segment fix-up sorts (unique keys, carried values).
//  k_fix_rows: one warp per CSR row, n <= 32 sorted in registers (shuffle
//              bitonic), then the sorted row is placed into the CSC.
//  k_fix_cols: one thread per CSC column, n <= kThreadCap sorted in place.
//  Longer segments go to k_sort_long (shared-memory rank sort, warp or block).
static constexpr int kThreadCap = 16;

__device__ __forceinline__ void warp_sort_regs(int& key, int& val, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      int pk = __shfl_xor_sync(0xffffffffu, key, j);
      int pv = __shfl_xor_sync(0xffffffffu, val, j);
      bool up = (lane & k) == 0;
      bool lower = (lane & j) == 0;
      bool take_min = lower == up;
      bool swap = take_min ? (pk < key) : (pk > key);
      if (swap) { key = pk; val = pv; }
    }
}

// Bitonic sort of 16 (key, value) pairs held by the 16 lanes of a half warp
// (hl = lane within the half); both halves of the warp sort independently.
__device__ __forceinline__ void half_sort_regs(int& key, int& val, int hl) {
#pragma unroll
  for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      int pk = __shfl_xor_sync(0xffffffffu, key, j);
      int pv = __shfl_xor_sync(0xffffffffu, val, j);
      bool up = (hl & k) == 0;
      bool lower = (hl & j) == 0;
      bool take_min = lower == up;
      bool swap = take_min ? (pk < key) : (pk > key);
      if (swap) { key = pk; val = pv; }
    }
}

__device__ __forceinline__ void place_sorted(int row, int b, int i, int key, int val,
                                             int* eperm, int* col, const int* col_ptr, int* ccur,
                                             int* csc_pos, int* csc_row) {
  eperm[b + i] = key;
  col[b + i] = val;
  if (col_ptr) {
    int w = col_ptr[val] + atomicAdd(&ccur[val], 1);
    csc_pos[w] = b + i;
    csc_row[w] = row;
  }
}

// Two rows per warp: a row of <= 16 entries is sorted by its half warp (10
// compare-exchange stages instead of 15 over a full warp); rows of 17..32 are
// then sorted one after another by the whole warp; longer rows go to
// k_sort_long.  Then the sorted row is placed into the CSC.
__global__ void __launch_bounds__(256)
k_fix_rows(int rows, const int* __restrict__ row_ptr, int* eperm, int* col,
           const int* __restrict__ col_ptr, int* ccur, int* csc_pos, int* csc_row, int* long_list,
           int* long_cnt) {
  const int lane = threadIdx.x & 31, hl = lane & 15;
  const int row0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 2;
  if (row0 >= rows) return;
  const int row = row0 + (lane >> 4);
  int b = 0, n = 0;
  if (row < rows) {
    b = row_ptr[row];
    n = row_ptr[row + 1] - b;
  }
  if (n > 32 && hl == 0) long_list[atomicAdd(long_cnt, 1)] = row;
  const bool small = n <= 16;
  int key = (small && hl < n) ? eperm[b + hl] : 0x7fffffff;
  int val = (small && hl < n) ? col[b + hl] : 0;
  if (__any_sync(0xffffffffu, small && n > 1)) half_sort_regs(key, val, hl);
  if (small && hl < n) place_sorted(row, b, hl, key, val, eperm, col, col_ptr, ccur, csc_pos, csc_row);
  unsigned mid = __ballot_sync(0xffffffffu, hl == 0 && n > 16 && n <= 32);
  while (mid) {
    const int src = __ffs(mid) - 1;
    mid &= mid - 1;
    const int bb = __shfl_sync(0xffffffffu, b, src), nn = __shfl_sync(0xffffffffu, n, src);
    const int rr = row0 + (src >> 4);
    int k2 = lane < nn ? eperm[bb + lane] : 0x7fffffff;
    int v2 = lane < nn ? col[bb + lane] : 0;
    warp_sort_regs(k2, v2, lane);
    if (lane < nn) place_sorted(rr, bb, lane, k2, v2, eperm, col, col_ptr, ccur, csc_pos, csc_row);
  }
}

// One warp per 32 consecutive CSC columns: lane l sorts column 32w+l in place
// when it has <= kThreadCap entries; columns of (kThreadCap, 32] are sorted by
// the whole warp in registers, one after another; longer ones go to the
// block-wide kernel.
__global__ void __launch_bounds__(256)
k_fix_cols(const int* __restrict__ U_dev, const int* __restrict__ col_ptr, int* csc_pos,
           int* csc_row, int* long_list, int* long_cnt) {
  const int lane = threadIdx.x & 31;
  const int U = *U_dev;
  const int u0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 32;
  if (u0 >= U) return;
  const int u = u0 + lane;
  int b = 0, n = 0;
  if (u < U) {
    b = col_ptr[u];
    n = col_ptr[u + 1] - b;
  }
  if (n > 1 && n <= kThreadCap) {
    // registers + odd-even transposition network (compile-time indices, no
    // dependent global-memory round trips)
    int kk[kThreadCap], vv[kThreadCap];
#pragma unroll
    for (int i = 0; i < kThreadCap; i++) {
      kk[i] = i < n ? csc_pos[b + i] : 0x7fffffff;
      vv[i] = i < n ? csc_row[b + i] : 0;
    }
#pragma unroll
    for (int ph = 0; ph < kThreadCap; ph++)
#pragma unroll
      for (int i = ph & 1; i + 1 < kThreadCap; i += 2)
        if (kk[i] > kk[i + 1]) {
          int t = kk[i]; kk[i] = kk[i + 1]; kk[i + 1] = t;
          t = vv[i]; vv[i] = vv[i + 1]; vv[i + 1] = t;
        }
#pragma unroll
    for (int i = 0; i < kThreadCap; i++)
      if (i < n) {
        csc_pos[b + i] = kk[i];
        csc_row[b + i] = vv[i];
      }
  }
  if (n > 32) long_list[atomicAdd(long_cnt, 1)] = u;
  unsigned mid = __ballot_sync(0xffffffffu, n > kThreadCap && n <= 32);
  while (mid) {
    const int src = __ffs(mid) - 1;
    mid &= mid - 1;
    const int bb = __shfl_sync(0xffffffffu, b, src), nn = __shfl_sync(0xffffffffu, n, src);
    int key = lane < nn ? csc_pos[bb + lane] : 0x7fffffff;
    int val = lane < nn ? csc_row[bb + lane] : 0;
    warp_sort_regs(key, val, lane);
    if (lane < nn) {
      csc_pos[bb + lane] = key;
      csc_row[bb + lane] = val;
    }
  }
}

// Segments longer than 32 (hub columns, long rows): rank sort in shared
// memory -- every key's final position is the number of smaller keys (keys
// are unique), computed with broadcast reads, no synchronisation chain.
// n <= kWarpRank: one warp per segment (8 per block); n <= kBlockRank: the
// whole block; longer (never seen in the workloads): rank sort in global.
static constexpr int kWarpRank = 256;
static constexpr int kBlockRank = 4096;

template <bool ROWS>
__device__ __forceinline__ void place_row_in_csc(int seg, int b, int e, int first, int step,
                                                 const int* vals, const int* col_ptr, int* ccur,
                                                 int* csc_pos, int* csc_row) {
  if (!ROWS || !col_ptr) return;
  for (int p = b + first; p < e; p += step) {
    const int c = vals[p];
    const int w = col_ptr[c] + atomicAdd(&ccur[c], 1);
    csc_pos[w] = p;
    csc_row[w] = seg;
  }
}

// Rank scatter: thread `t` of `nt` owns keys t, t+nt, ... (at most E, held in
// registers); every key of the segment is read once per thread with 16-byte
// shared loads (broadcast) and compared against all owned keys, so one load
// serves 4*E comparisons.  The segment buffer is padded to a multiple of 4
// with INT_MAX by the caller.
template <int E>
__device__ __forceinline__ void rank_scatter(const int* sk, const int* sv, int n, int t, int nt,
                                             int* keys, int* vals) {
  int kk[E], r[E];
#pragma unroll
  for (int q = 0; q < E; q++) {
    const int i = t + q * nt;
    kk[q] = i < n ? sk[i] : 0x7fffffff;
    r[q] = 0;
  }
  const int n4 = (n + 3) >> 2;
  for (int j = 0; j < n4; j++) {
    const int4 v = reinterpret_cast<const int4*>(sk)[j];
#pragma unroll
    for (int q = 0; q < E; q++)
      r[q] += (v.x < kk[q]) + (v.y < kk[q]) + (v.z < kk[q]) + (v.w < kk[q]);
  }
#pragma unroll
  for (int q = 0; q < E; q++) {
    const int i = t + q * nt;
    if (i < n) {
      keys[r[q]] = kk[q];
      vals[r[q]] = sv[i];
    }
  }
}

static constexpr int kSortThreads = 512;

template <bool ROWS>
__global__ void __launch_bounds__(kSortThreads)
k_sort_long(const int* __restrict__ ptr, int* keys, int* vals, const int* __restrict__ col_ptr,
            int* ccur, int* csc_pos, int* csc_row, const int* list, const int* cnt, int* gk,
            int* gv, int dbg) {
  constexpr int NW = kSortThreads / 32;
  static_assert(NW * kWarpRank <= kBlockRank, "warp slices must fit the block buffer");
  __shared__ __align__(16) int sk[kBlockRank];
  __shared__ __align__(16) int sv[kBlockRank];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n_long = *cnt;
  // ---- warp phase (32 < n <= kWarpRank)
  int* wk = sk + w * kWarpRank;
  int* wv = sv + w * kWarpRank;
  for (int k = blockIdx.x * NW + w; k < n_long; k += gridDim.x * NW) {
    const int seg = list[k];
    const int b = ptr[seg], e = ptr[seg + 1], n = e - b;
    if (n > kWarpRank || (dbg & 1)) continue;
    for (int i = lane; i < ((n + 3) & ~3); i += 32) {
      wk[i] = i < n ? keys[b + i] : 0x7fffffff;
      wv[i] = i < n ? vals[b + i] : 0;
    }
    __syncwarp();
    rank_scatter<kWarpRank / 32>(wk, wv, n, lane, 32, keys + b, vals + b);
    __syncwarp();
    place_row_in_csc<ROWS>(seg, b, e, lane, 32, vals, col_ptr, ccur, csc_pos, csc_row);
  }
  __syncthreads();
  // ---- block phase (n > kWarpRank): one segment per block, shared memory
  // rank sort up to kBlockRank, global-memory rank sort beyond
  for (int k = blockIdx.x; k < n_long; k += gridDim.x) {
    const int seg = list[k];
    const int b = ptr[seg], e = ptr[seg + 1], n = e - b;
    if (n <= kWarpRank || (dbg & 2)) continue;
    if (n <= kBlockRank) {
      // bitonic sort in shared memory, padded to a power of two
      int P = 1;
      while (P < n) P <<= 1;
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        sk[i] = i < n ? keys[b + i] : 0x7fffffff;
        sv[i] = i < n ? vals[b + i] : 0;
      }
      __syncthreads();
      for (int kk = 2; kk <= P; kk <<= 1)
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
            // i-th compare-exchange pair of this stage
            const int lo = ((i / jj) * 2 * jj) + (i % jj), hi = lo + jj;
            const bool up = (lo & kk) == 0;
            const int a = sk[lo], c = sk[hi];
            if ((a > c) == up) {
              sk[lo] = c; sk[hi] = a;
              const int t = sv[lo]; sv[lo] = sv[hi]; sv[hi] = t;
            }
          }
          __syncthreads();
        }
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        keys[b + i] = sk[i];
        vals[b + i] = sv[i];
      }
    } else {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        gk[b + i] = keys[b + i];
        gv[b + i] = vals[b + i];
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int kk = gk[b + i];
        int r = 0;
        for (int j = 0; j < n; j++) r += gk[b + j] < kk;
        keys[b + r] = kk;
        vals[b + r] = gv[b + i];
      }
    }
    __syncthreads();
    place_row_in_csc<ROWS>(seg, b, e, threadIdx.x, blockDim.x, vals, col_ptr, ccur, csc_pos,
                           csc_row);
    __syncthreads();
  }
}

struct BuildWs {
  int *cnt, *pre, *key_e, *slot_e, *cur, *ccnt, *ccur, *scan, *lists, *counters, *gk, *gv;
};

static size_t build_ws(const LayerMeta& m, long long U_max, char* base, BuildWs* w) {
  long long nz = (long long)m.rows + m.S;
  long long sc = (long long)scan_ws_ints(nz > U_max ? nz : U_max);
  size_t b = 0;
  b += carve_bytes(nz, 4);              // cnt
  b += carve_bytes(nz + 1, 4);          // pre
  b += carve_bytes(m.N, 4) * 2;         // key_e, slot_e
  b += carve_bytes(m.rows, 4);          // cur
  b += carve_bytes(U_max + 1, 4) * 2;   // ccnt, ccur
  b += carve_bytes(sc, 4);              // scan
  b += carve_bytes((long long)m.rows + U_max, 4);  // long lists
  b += carve_bytes(2, 4);               // counters
  b += carve_bytes(m.N, 4) * 2;         // gk, gv
  if (base && w) {
    char* p = base;
    w->cnt = carve<int>(p, nz);
    w->pre = carve<int>(p, nz + 1);
    w->key_e = carve<int>(p, m.N);
    w->slot_e = carve<int>(p, m.N);
    w->cur = carve<int>(p, m.rows);
    w->ccnt = carve<int>(p, U_max + 1);
    w->ccur = carve<int>(p, U_max + 1);
    w->scan = carve<int>(p, sc);
    w->lists = carve<int>(p, (long long)m.rows + U_max);
    w->counters = carve<int>(p, 2);
    w->gk = carve<int>(p, m.N);
    w->gv = carve<int>(p, m.N);
  }
  return b;
}

static long long umax_of(const LayerMeta& m) { return m.N < m.S ? m.N : m.S; }

}  // namespace hf

using namespace hf;

extern "C" {

hifuse_status hifuse_csr_sizes(const hifuse_layer_shape* shape, hifuse_layout layout,
                               int64_t* rows, int64_t* U_max, int64_t* S, size_t* ws_bytes) {
  if (layout != HIFUSE_LAYOUT_COMPACT) return HIFUSE_ERR_UNSUPPORTED;
  LayerMeta m;
  hifuse_status st = make_meta(shape, &m);
  if (st != HIFUSE_OK) return st;
  if (rows) *rows = m.rows;
  if (U_max) *U_max = umax_of(m);
  if (S) *S = m.S;
  if (ws_bytes) *ws_bytes = build_ws(m, umax_of(m), nullptr, nullptr);
  return HIFUSE_OK;
}

hifuse_status hifuse_build_semantic_graphs(const hifuse_layer_shape* shapes, int num_layers,
                                           const int32_t* const* d_src_local,
                                           const int32_t* const* d_dst_local,
                                           const int64_t* const* d_edge_id,
                                           const int32_t* d_edge_type, int64_t num_graph_edges,
                                           const int64_t* d_rel_edge_off,
                                           hifuse_layout layout, const hifuse_csr* out,
                                           void* d_ws, size_t ws_bytes, int32_t* d_status,
                                           hifuse_stream_t stream) {
  if (layout != HIFUSE_LAYOUT_COMPACT) return HIFUSE_ERR_UNSUPPORTED;
  if (!shapes || num_layers <= 0 || !d_src_local || !d_dst_local || !d_edge_id || !out ||
      !d_status || num_graph_edges < 0 ||
      (num_graph_edges > 0 && !d_edge_type && !d_rel_edge_off))
    return HIFUSE_ERR_INVALID_ARG;
  cudaStream_t s = st(stream);
  static const int dbg = getenv("HIFUSE_DBG_SORT") ? atoi(getenv("HIFUSE_DBG_SORT")) : 0;
  std::vector<LayerMeta> metas(num_layers);
  LayerMeta* mv = metas.data();
  hifuse_status rc = HIFUSE_OK;
  for (int l = 0; l < num_layers && rc == HIFUSE_OK; l++) {
    rc = make_meta(&shapes[l], &mv[l]);
    if (rc != HIFUSE_OK) break;
    const hifuse_csr& o = out[l];
    if (!o.rel_row_off || !o.row_ptr || !o.rel_y_off || !o.U_dev ||
        (mv[l].N > 0 && (!d_src_local[l] || !d_dst_local[l] || !d_edge_id[l] || !o.col ||
                         !o.eperm || !o.y_src)) ||
        (!o.col_ptr != !o.csc_pos || !o.col_ptr != !o.csc_row) ||
        (mv[l].S > 0 && !o.slot_y))
      rc = HIFUSE_ERR_INVALID_ARG;
    else if (build_ws(mv[l], umax_of(mv[l]), nullptr, nullptr) > ws_bytes || !d_ws)
      rc = HIFUSE_ERR_WORKSPACE;
  }
  if (rc != HIFUSE_OK) return rc;
  for (int l = 0; l < num_layers; l++) {
    const LayerMeta& m = mv[l];
    const hifuse_csr& o = out[l];
    long long U_max = umax_of(m);
    BuildWs w;
    build_ws(m, U_max, (char*)d_ws, &w);
    long long nz = (long long)m.rows + m.S;
    cudaMemsetAsync(w.cnt, 0, sizeof(int) * (nz > 0 ? nz : 1), s);
    cudaMemsetAsync(w.cur, 0, sizeof(int) * (m.rows > 0 ? m.rows : 1), s);
    // the transpose (CSC) is optional: a layer whose aggregation backward is
    // never run (the input layer of the aggregate-first RGCN) passes NULLs
    const bool csc = o.col_ptr != nullptr;
    if (csc) {
      cudaMemsetAsync(w.ccnt, 0, sizeof(int) * (U_max + 1), s);
      cudaMemsetAsync(w.ccur, 0, sizeof(int) * (U_max + 1), s);
    }
    cudaMemsetAsync(w.counters, 0, sizeof(int) * 2, s);
    const int TB = 256;
    HF_LAUNCH(k_classify, ceil_div(m.N, TB), TB, 0, s, m, d_src_local[l], d_dst_local[l],
              (const long long*)d_edge_id[l], d_edge_type, (const long long*)d_rel_edge_off,
              (long long)num_graph_edges, w.key_e,
              w.slot_e, w.cnt, d_status);
    exclusive_scan(w.cnt, w.pre, nz, w.scan, s);
    long long fin = nz + 1 > m.R + 1 ? nz + 1 : m.R + 1;
    HF_LAUNCH(k_finish, ceil_div(fin, TB), TB, 0, s, m, w.cnt, w.pre, o.row_ptr, o.rel_row_off,
              o.rel_y_off, o.y_src, o.slot_y, o.U_dev);
    HF_LAUNCH(k_scatter, ceil_div(m.N, TB), TB, 0, s, m, w.key_e, w.slot_e, o.row_ptr, o.slot_y,
              w.cur, w.ccnt, o.eperm, o.col, o.csc_pos, o.csc_row);
    if (csc) exclusive_scan(w.ccnt, o.col_ptr, U_max, w.scan, s);
    int* rows_long = w.lists;
    int* cols_long = w.lists + m.rows;
    HF_LAUNCH(k_fix_rows, ceil_div(m.rows, 16), 256, 0, s, m.rows, o.row_ptr, o.eperm, o.col,
              o.col_ptr, w.ccur, o.csc_pos, o.csc_row, rows_long, w.counters);
    HF_LAUNCH(k_sort_long<true>, 148, kSortThreads, 0, s, o.row_ptr, o.eperm, o.col, o.col_ptr, w.ccur,
              o.csc_pos, o.csc_row, rows_long, w.counters, w.gk, w.gv, dbg);
    if (!csc) continue;
    HF_LAUNCH(k_fix_cols, ceil_div(U_max, 256), 256, 0, s, o.U_dev, o.col_ptr, o.csc_pos,
              o.csc_row, cols_long, w.counters + 1);   // 8 warps x 32 columns per block
    HF_LAUNCH(k_sort_long<false>, 148, kSortThreads, 0, s, o.col_ptr, o.csc_pos, o.csc_row,
              (const int*)nullptr, (int*)nullptr, (int*)nullptr, (int*)nullptr, cols_long,
              w.counters + 1, w.gk, w.gv, dbg);
  }
  return last_cuda();
}

hifuse_status hifuse_edge_type_offsets(const int32_t* d_edge_type, int64_t num_graph_edges,
                                       int num_rels, int64_t* d_rel_edge_off, int32_t* d_status,
                                       hifuse_stream_t stream) {
  if (num_graph_edges < 0 || num_rels <= 0 || num_rels > HF_MAX_R || !d_rel_edge_off ||
      !d_status || (num_graph_edges > 0 && !d_edge_type))
    return HIFUSE_ERR_INVALID_ARG;
  cudaStream_t s = st(stream);
  if (num_graph_edges > 0)
    HF_LAUNCH(k_et_check, ceil_div(num_graph_edges, 256), 256, 0, s, d_edge_type,
              (long long)num_graph_edges, num_rels, d_status);
  HF_LAUNCH(k_et_offsets, ceil_div(num_rels + 1, 64), 64, 0, s, d_edge_type,
            (long long)num_graph_edges, num_rels, (long long*)d_rel_edge_off);
  return last_cuda();
}

}  // extern "C"

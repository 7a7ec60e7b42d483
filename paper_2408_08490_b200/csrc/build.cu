// build.cu -- A1: semantic graph build (Alg. 2) as a
// merged segmented CSR + CSC for EVERY layer of a step in six launches (one
// memset + five kernels), independent of the number of relations R and of
// the number of layers.
//
// Alg. 2 runs, per layer, 1 gather (line 316) + R compares (318) + R
// index-selects (319): 2R+1 short kernels that the paper offloads to the CPU
// (lines 299-336; "numerous and short", line 174).  Here the relation of an
// edge only decides a KEY,
//   key(e) = rel_row_off[r(e)] + dst(e)      (merged row, relation-major),
// and one counting sort by key performs every relation's selection at once.
// Every kernel covers all layers of the call (a flattened (layer, tile) grid):
//   memset      per-layer counters (one contiguous zone)
//   k_classify  EdgeTypeLayer (gather, or binary search of relation-major
//               edge-id ranges) + validation; row histogram (warp-aggregated
//               reductions: one per distinct row of a warp); per (relation,
//               source) slot the number of edges
//   k_scan      segmented decoupled-look-back scan of the row counts and of
//               the slot (presence, count) pairs: row_ptr, rel_row_off,
//               slot_y, y_src, rel_y_off, U -- and col_ptr, because Y rows are
//               numbered in slot order, so the CSC column of Y row slot_y[s]
//               starts at the exclusive prefix of the slot counts at s
//               Also the runs of each row (stretches of consecutive input
//               edges with one key) and the first edge of a run
//   k_scatter   pos = row_ptr[key] + (e - first edge of the run) for a row of
//               ONE run (input order: the sampler lists a destination's edges
//               of a relation together), else + an arrival ticket (unsorted):
//               eperm, col.  (k_classify's row histogram is therefore a
//               fire-and-forget reduction: no atomic round trip per edge.)
//   k_rows      warp per HF_BUILD_ROWS_PER_WARP consecutive rows: their CSR
//               span staged in shared memory, every row of several runs sorted
//               by original column (restores Alg. 2's order: bit-exact and
//               deterministic), then placed into the
//               CSC (one atomic slot per entry); longer rows by the block
//   k_cols      warp per 32 consecutive CSC columns: each sorted by CSR
//               position (lane per column <= 16 entries, warp bitonic <= 32),
//               hub columns by a warp (rank) / the block (bitonic) in smem
// The kernels are short with many blocks, so on the pipelined step (build of
// batch i+1 on a low-priority side stream) they interleave with the compute
// of batch i at block granularity.  (A single persistent kernel with
// ticket-ordered phases was measured and dropped: resident for the whole
// build, it starved the compute stream -- DESIGN.md §8.)
#include <algorithm>
#include <cstring>
#include <vector>
#include "common.cuh"

namespace hf {

namespace {

constexpr int kBT = 256;               // threads per block
constexpr int kNW = kBT / 32;
// Tiling (compile-time; scripts/build_variants.sh + scripts/sweep_build.py
// sweep them).  Measured on B200 (eager build call, mag / IMDB / Freebase /
// DBLP): 2048 edges per block, 16 scan elements per thread, 32 rows per warp
// -> 75 / 62 / 76 / 74 us; 512 / 4 / 8 -> 62 / 46 / 67 / 53 us: the kernels
// are latency-bound, so more, smaller blocks (more warps in flight) win.
#ifndef HF_BUILD_EDGE_TILE
#define HF_BUILD_EDGE_TILE 512
#endif
#ifndef HF_BUILD_SCAN_PER
#define HF_BUILD_SCAN_PER 4
#endif
#ifndef HF_BUILD_ROWS_PER_WARP
#define HF_BUILD_ROWS_PER_WARP 8
#endif
constexpr int kEdgeTile = HF_BUILD_EDGE_TILE;   // edges per classify / scatter block
constexpr int kEPT = kEdgeTile / kBT;  // edges per thread
constexpr int kScanPer = HF_BUILD_SCAN_PER;   // scan elements per thread
constexpr int kScanTile = kBT * kScanPer;
constexpr int kSegRows = 32;           // rows / columns per warp in k_rows / k_cols
constexpr int kSegTile = kNW * kSegRows;
constexpr int kRowsW = HF_BUILD_ROWS_PER_WARP;  // merged rows per warp in k_rows
constexpr int kRowsTile = kNW * kRowsW;
constexpr int kSpanR = kRowsW * 32 < 1024 ? kRowsW * 32 : 1024;   // k_rows staging per warp
constexpr int kBlockRankR = kRowsW >= 16 ? 4096 : 2048;           // k_rows long-row sort
constexpr size_t kSmemRows = (size_t)(kNW * kSpanR * 2 > 2 * kBlockRankR ? kNW * kSpanR * 2
                                                                        : 2 * kBlockRankR) *
                             sizeof(int);
constexpr int kSpan = 1024;            // CSR/CSC entries a warp stages in smem
constexpr int kMaxL = 4;               // layers per launch set (more: further sets)
constexpr int kWarpRank = 256;
constexpr int kBlockRank = 4096;
constexpr int kLongRowBlocks = 16;     // k_rows blocks for rows > 32 (not in workloads)
constexpr size_t kSmem = (size_t)kNW * kSpan * 2 * sizeof(int);   // 64 KB
static_assert(kBlockRank * 2 * sizeof(int) <= kSmem, "block rank sort buffer");
constexpr size_t kSmemScan = 2 * (kScanTile + kScanTile / 32) * sizeof(int) + 128;
static_assert(kSmemScan <= kSmem, "scan buffer");

enum Kern { K_CLASSIFY, K_SCAN, K_SCATTER, K_ROWS, K_COLS, kKerns };

struct BLayer {
  int R, N, rows, S, U_max, csc;
  int ynum;                            // 0: X-row columns (no Y numbering, no slots)
  int t_rows, t_slots;                 // scan tiles per segment
  int key_base[HF_MAX_R + 1];          // rel_row_off
  int slot_base[HF_MAX_R + 1];         // slot_off
  int src_lim[HF_MAX_R];               // n_src of the source type of r
  int xoff[HF_MAX_R];                  // type_src_off of the source type of r (X-row mode)
  int dst_lim[HF_MAX_R];               // n_dst of the destination type of r
  const int* src;
  const int* dst;
  const long long* eid;
  // outputs
  int *o_rel_row_off, *row_ptr, *col, *eperm, *o_rel_y_off, *y_src, *col_ptr, *csc_pos,
      *csc_row, *csc_col, *slot_y, *U_dev;
  const int* xg;                       // X-row mode: feature-store row of every X row
  // workspace: zero zone
  int *cnt, *ccur;                     // cnt = [row counts | slot counts]
  int* runs;                           // per row: runs of consecutive input edges
  int* rcur;                           // per row: arrival tickets (rows of several runs)
  int* lcnt;                           // [0] long rows, [1] long columns
  unsigned long long* sst;             // scan tile status [t_rows | t_slots]
  // workspace: scratch
  int *key_e, *slot_e, *gk, *gv, *long_rows, *long_cols;
  int* first;                          // per row: first input edge of its (last) run
  int rows_reg, cols_reg;              // regular (non-long) blocks of k_rows / k_cols
  int cols_xtra;                       // extra k_cols blocks for hub columns
};

struct BPlan {
  int L;
  int blk_off[kKerns][kMaxL + 1];      // block ranges of the layers in each kernel
  long long E;
  const int* edge_type;
  const long long* rel_off;
  int* status;
};

struct BuildParams {
  BPlan p;
  BLayer lay[kMaxL];
};
static_assert(sizeof(BuildParams) <= 32764, "kernel parameter space (32 KB)");

// (layer, tile) of this block in kernel k
__device__ __forceinline__ int layer_of(const BPlan& P, int k, int* j) {
  const int b = blockIdx.x;
  int l = 0;
  while (l + 1 < P.L && b >= P.blk_off[k][l + 1]) l++;
  *j = b - P.blk_off[k][l];
  return l;
}

// ------------------------------------------------------------ primitives --
// Look-back polls use relaxed loads (an acquire load per poll compiles to an
// L1 invalidation that stalls every block on the SM); the tile statuses are
// themselves the data.
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void warp_sort_regs(int& key, int& val, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      int pk = __shfl_xor_sync(0xffffffffu, key, j);
      int pv = __shfl_xor_sync(0xffffffffu, val, j);
      bool up = (lane & k) == 0;
      bool lower = (lane & j) == 0;
      bool swap = (lower == up) ? (pk < key) : (pk > key);
      if (swap) { key = pk; val = pv; }
    }
}

// bitonic sort of the 16 (key, value) pairs of each half warp (hl = lane & 15)
__device__ __forceinline__ void half_sort_regs(int& key, int& val, int hl) {
#pragma unroll
  for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      int pk = __shfl_xor_sync(0xffffffffu, key, j);
      int pv = __shfl_xor_sync(0xffffffffu, val, j);
      bool up = (hl & k) == 0;
      bool lower = (hl & j) == 0;
      bool swap = (lower == up) ? (pk < key) : (pk > key);
      if (swap) { key = pk; val = pv; }
    }
}

// Rank sort of n unique keys (+ values) held in shared memory (sk, sv, padded
// with INT_MAX to a multiple of 4): thread t of nt owns keys t, t+nt, ...;
// every key's final position is the number of smaller keys.
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

// Copies n entries of two int arrays into shared memory, 8 loads per thread
// in flight before the stores; [n, pad) is filled with (INT_MAX, 0).
__device__ __forceinline__ void stage2(const int* __restrict__ ka, const int* __restrict__ va,
                                       int n, int pad, int* sk, int* sv, int t, int nt) {
  constexpr int B = 8;
  for (int i0 = 0; i0 < pad; i0 += B * nt) {
    int kk[B], vv[B];
#pragma unroll
    for (int q = 0; q < B; q++) {
      const int i = i0 + q * nt + t;
      kk[q] = i < n ? ka[i] : 0x7fffffff;
      vv[q] = i < n ? va[i] : 0;
    }
#pragma unroll
    for (int q = 0; q < B; q++) {
      const int i = i0 + q * nt + t;
      if (i < pad) {
        sk[i] = kk[q];
        sv[i] = vv[q];
      }
    }
  }
}

// CSC placement of CSR position p (row `row`, Y row c)
__device__ __forceinline__ void place_entry(const BLayer& L, int row, int p, int c) {
  const int w = L.col_ptr[c] + atomicAdd(L.ccur + c, 1);
  L.csc_pos[w] = p;
  L.csc_row[w] = row;
  L.csc_col[w] = c;
}

// Block-wide sort of one segment [b, e) of (keys, vals): rank sort in shared
// memory (<= BR entries), a global rank sort beyond (never seen in the
// workloads).  sm: >= 2 BR ints.  Ends with __syncthreads.
template <int BR>
__device__ void block_sort_segment(int* keys, int* vals, int b, int e, int* sm, int* gk,
                                   int* gv) {
  const int n = e - b;
  int* sk = sm;
  int* sv = sm + BR;
  if (n <= BR) {
    // bitonic sort in shared memory, padded to a power of two (n log^2 n;
    // a rank sort is n^2 -- 30 us for a 1757-entry hub column of ogbn-mag)
    int P2 = 1;
    while (P2 < n) P2 <<= 1;
    stage2(keys + b, vals + b, n, P2, sk, sv, threadIdx.x, kBT);
    __syncthreads();
    for (int kk = 2; kk <= P2; kk <<= 1)
      for (int jj = kk >> 1; jj > 0; jj >>= 1) {
        for (int i = threadIdx.x; i < P2 / 2; i += kBT) {
          const int lo = ((i / jj) * 2 * jj) + (i % jj), hi = lo + jj;
          const bool up = (lo & kk) == 0;
          const int x = sk[lo], y = sk[hi];
          if ((x > y) == up) {
            sk[lo] = y; sk[hi] = x;
            const int tv = sv[lo]; sv[lo] = sv[hi]; sv[hi] = tv;
          }
        }
        __syncthreads();
      }
    for (int i = threadIdx.x; i < n; i += kBT) {
      keys[b + i] = sk[i];
      vals[b + i] = sv[i];
    }
  } else {
    for (int i = threadIdx.x; i < n; i += kBT) {
      gk[b + i] = keys[b + i];
      gv[b + i] = vals[b + i];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kBT) {
      const int kk = gk[b + i];
      int r = 0;
      for (int q = 0; q < n; q++) r += gk[b + q] < kk;
      keys[b + r] = kk;
      vals[b + r] = gv[b + i];
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------- k_classify --
struct RelSmem {
  long long off[HF_MAX_R + 1];         // relation-major edge-id ranges
  int key_base[HF_MAX_R + 1], slot_base[HF_MAX_R + 1], src_lim[HF_MAX_R], dst_lim[HF_MAX_R];
  int xoff[HF_MAX_R];
};

// Merged-row key of input edge e, -3 if the edge is invalid (k_classify's
// per-edge logic for a single edge: the one before a tile).
__device__ int edge_key_of(const BPlan& P, const BLayer& L, const RelSmem& rs, int e) {
  const long long id = L.eid[e];
  if (id < 0 || id >= P.E) return -3;
  int r;
  if (P.rel_off) {
    int lo = 0, hi = L.R;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rs.off[mid] <= id) lo = mid; else hi = mid;
    }
    r = lo;
  } else {
    r = P.edge_type[id];
  }
  if (r < 0 || r >= L.R) return -3;
  const int sv = L.src[e], dv = L.dst[e];
  if (sv < 0 || sv >= rs.src_lim[r] || dv < 0 || dv >= rs.dst_lim[r]) return -3;
  return rs.key_base[r] + dv;
}

__global__ void __launch_bounds__(kBT)
k_classify(const __grid_constant__ BuildParams bp) {
  HF_PDL_ENTRY();
  __shared__ RelSmem rs;
  __shared__ int skey[kEdgeTile];
  __shared__ int s_prev0;
  const BPlan& P = bp.p;
  int j;
  const BLayer& L = bp.lay[layer_of(P, K_CLASSIFY, &j)];
  // per-relation tables in shared memory (divergent relation ids would
  // serialise constant-bank reads of the kernel parameters)
  for (int i = threadIdx.x; i <= L.R; i += kBT) {
    if (P.rel_off) rs.off[i] = P.rel_off[i];
    rs.key_base[i] = L.key_base[i];
    rs.slot_base[i] = L.slot_base[i];
    if (i < L.R) {
      rs.src_lim[i] = L.src_lim[i];
      rs.dst_lim[i] = L.dst_lim[i];
      rs.xoff[i] = L.xoff[i];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int e0 = j * kEdgeTile;
  long long id[kEPT];
  int sv[kEPT], dv[kEPT], key[kEPT], slot[kEPT];
  // all loads of the thread in flight together
#pragma unroll
  for (int q = 0; q < kEPT; q++) {
    const int e = e0 + q * kBT + threadIdx.x;
    const bool in = e < L.N;
    id[q] = in ? L.eid[e] : -2;
    sv[q] = in ? L.src[e] : 0;
    dv[q] = in ? L.dst[e] : 0;
  }
  int bad_any = 0;
#pragma unroll
  for (int q = 0; q < kEPT; q++) {
    key[q] = -1;
    slot[q] = -1;
    if (id[q] == -2) continue;                     // past the tile
    if (id[q] == -1) {                             // null (padding) edge: dropped silently
      key[q] = -3;
      continue;
    }
    int bad = 0, r = -1;
    if (id[q] < 0 || id[q] >= P.E) {
      bad = HIFUSE_ST_BAD_EDGE_ID;
    } else {
      // Alg. 2: EdgeTypeLayer = EdgeType[EdgeID] -- a gather, or for
      // a relation-major table the relation whose id range holds `id`
      if (P.rel_off) {
        int lo = 0, hi = L.R;                       // off[lo] <= id < off[hi]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (rs.off[mid] <= id[q]) lo = mid; else hi = mid;
        }
        r = lo;
      } else {
        r = P.edge_type[id[q]];
      }
      if (r < 0 || r >= L.R) bad = HIFUSE_ST_BAD_REL;
      else if (sv[q] < 0 || sv[q] >= rs.src_lim[r]) bad = HIFUSE_ST_BAD_SRC;
      else if (dv[q] < 0 || dv[q] >= rs.dst_lim[r]) bad = HIFUSE_ST_BAD_DST;
    }
    if (bad) {
      bad_any |= bad;
      key[q] = -3;                                 // dropped edge
      continue;
    }
    key[q] = rs.key_base[r] + dv[q];               // lines 318-319, every r at once
    // Y numbering: the (relation, source) slot (index into cnt); X-row mode:
    // the source's row in the layer's type-major X (the column itself)
    slot[q] = L.ynum ? L.rows + rs.slot_base[r] + sv[q] : rs.xoff[r] + sv[q];
  }
  if (bad_any) atomicOr(P.status, bad_any);
  // Runs: maximal stretches of consecutive valid input edges with one key.  A
  // row made of ONE run (sampled blocks list a destination's edges of one
  // relation together) is placed in input order by k_scatter directly
  // (position = e - first edge of the run) and needs no sort in k_rows.
#pragma unroll
  for (int q = 0; q < kEPT; q++) skey[q * kBT + threadIdx.x] = key[q];
  if (threadIdx.x == 0) s_prev0 = e0 > 0 ? edge_key_of(P, L, rs, e0 - 1) : -1;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kEPT; q++) {
    const int i = q * kBT + threadIdx.x;
    const int prev = i ? skey[i - 1] : s_prev0;
    if (key[q] >= 0 && prev != key[q]) {
      L.first[key[q]] = e0 + i;
      atomicAdd(L.runs + key[q], 1);
    }
  }
  // Warp-aggregated atomics: sampled blocks list the edges of a destination
  // (and often of a source) together, so lanes of a warp often share a row
  // or slot -- one atomic per distinct address and warp.
  unsigned prow[kEPT], pslot[kEPT];
#pragma unroll
  for (int q = 0; q < kEPT; q++) {
    prow[q] = __match_any_sync(0xffffffffu, key[q] >= 0 ? key[q] : -1 - lane);
    pslot[q] = L.ynum ? __match_any_sync(0xffffffffu, key[q] >= 0 ? slot[q] : -1 - lane) : 0u;
  }
  // counts only (no return value: fire-and-forget reductions); an edge's
  // position inside its row is formed by k_scatter -- from its run for a row
  // of one run, from an arrival ticket for the (rare) rows of several runs
#pragma unroll
  for (int q = 0; q < kEPT; q++) {
    const bool lead_r = key[q] >= 0 && lane == __ffs(prow[q]) - 1;
    const bool lead_s = L.ynum && key[q] >= 0 && lane == __ffs(pslot[q]) - 1;
    if (lead_r) atomicAdd(L.cnt + key[q], __popc(prow[q]));
    if (lead_s) atomicAdd(L.cnt + slot[q], __popc(pslot[q]));
  }
#pragma unroll
  for (int q = 0; q < kEPT; q++) {
    const int e = e0 + q * kBT + threadIdx.x;
    if (key[q] == -1) continue;
    L.key_e[e] = key[q] >= 0 ? key[q] : -1;
    if (key[q] >= 0) L.slot_e[e] = L.ynum ? slot[q] - L.rows : slot[q];
  }
}

// ----------------------------------------------------------------- k_scan --
// Segmented exclusive scan, decoupled look-back over the tiles of a segment.
// Rows segment: the row counts.  Slots segment: (presence, count) pairs of
// the (relation, source) slots -- presence numbers the Y rows (slot_y,
// y_src, rel_y_off, U), the counts give col_ptr.  Tile status (u64):
// flag << 62 | a << 31 | b, flag 1 aggregate, 2 inclusive prefix; a, b < 2^31.
constexpr unsigned long long kValMask = (1ull << 31) - 1;

__device__ __forceinline__ unsigned long long pack(int flag, long long a, long long b) {
  return ((unsigned long long)flag << 62) | ((unsigned long long)a << 31) | (unsigned long long)b;
}

__global__ void __launch_bounds__(kBT)
k_scan(const __grid_constant__ BuildParams bp) {
  HF_PDL_ENTRY();
  extern __shared__ __align__(16) int sm[];
  int jj;
  const BLayer& L = bp.lay[layer_of(bp.p, K_SCAN, &jj)];
  const bool rows_seg = jj < L.t_rows;
  const int j = rows_seg ? jj : jj - L.t_rows;
  const int* a = rows_seg ? L.cnt : L.cnt + L.rows;
  const int len = rows_seg ? L.rows : L.S;
  unsigned long long* st = rows_seg ? L.sst : L.sst + L.t_rows;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int base = j * kScanTile;
  const int n = max(0, min(kScanTile, len - base));
  int* buf = sm;                                    // counts, then count prefixes
  int* fbuf = sm + kScanTile + kScanTile / 32;      // flag prefixes (slots)
  __shared__ int wsum[2 * kNW];
  __shared__ long long s_pre[2];
  auto pad = [](int i) { return i + (i >> 5); };
  // coalesced load, 16 per thread in flight
  {
    int v[kScanPer];
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
      const int i = k * kBT + t;
      v[k] = i < n ? a[base + i] : 0;
    }
#pragma unroll
    for (int k = 0; k < kScanPer; k++) buf[pad(k * kBT + t)] = v[k];
  }
  __syncthreads();
  int c[kScanPer];
  int csum = 0, fsum = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; k++) {
    c[k] = buf[pad(t * kScanPer + k)];
    csum += c[k];
    fsum += c[k] > 0;
  }
  // block exclusive scan of the per-thread (count, flag) sums
  int ci = csum, fi = fsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y1 = __shfl_up_sync(0xffffffffu, ci, o);
    const int y2 = __shfl_up_sync(0xffffffffu, fi, o);
    if (lane >= o) { ci += y1; fi += y2; }
  }
  if (lane == 31) { wsum[w] = ci; wsum[kNW + w] = fi; }
  __syncthreads();
  if (w == 0) {
    int x1 = lane < kNW ? wsum[lane] : 0, x2 = lane < kNW ? wsum[kNW + lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y1 = __shfl_up_sync(0xffffffffu, x1, o);
      const int y2 = __shfl_up_sync(0xffffffffu, x2, o);
      if (lane >= o) { x1 += y1; x2 += y2; }
    }
    if (lane < kNW) { wsum[lane] = x1; wsum[kNW + lane] = x2; }
  }
  __syncthreads();
  const int cex = (w ? wsum[w - 1] : 0) + ci - csum;
  const int fex = (w ? wsum[kNW + w - 1] : 0) + fi - fsum;
  const long long cagg = wsum[kNW - 1], fagg = wsum[2 * kNW - 1];
  // look-back (warp 0)
  if (w == 0) {
    long long ce = 0, fe = 0;
    if (j == 0) {
      if (lane == 0) st_release64(st, pack(2, fagg, cagg));
    } else {
      if (lane == 0) st_release64(st + j, pack(1, fagg, cagg));
      int k = j - 1;
      for (;;) {
        const int idx = k - lane;
        unsigned long long sv;
        for (int ns = 32;; ns = min(ns * 2, 256)) {
          sv = idx >= 0 ? ld_relaxed64(st + idx) : pack(2, 0, 0);
          if (__all_sync(0xffffffffu, (sv >> 62) != 0)) break;
          __nanosleep(ns);
        }
        const unsigned incl = __ballot_sync(0xffffffffu, (sv >> 62) == 2);
        const int stop = incl ? __ffs(incl) - 1 : 31;
        long long va = lane <= stop ? (long long)((sv >> 31) & kValMask) : 0;
        long long vb = lane <= stop ? (long long)(sv & kValMask) : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          va += __shfl_xor_sync(0xffffffffu, va, o);
          vb += __shfl_xor_sync(0xffffffffu, vb, o);
        }
        fe += va;
        ce += vb;
        if (incl) break;
        k -= 32;
      }
      if (lane == 0) st_release64(st + j, pack(2, fe + fagg, ce + cagg));
    }
    if (lane == 0) { s_pre[0] = ce; s_pre[1] = fe; }
  }
  __syncthreads();
  const long long cpre = s_pre[0], fpre = s_pre[1];
  const bool last_tile = base + kScanTile >= len;
  long long crun = cpre + cex, frun = fpre + fex;
  if (rows_seg) {
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
      buf[pad(t * kScanPer + k)] = (int)crun;
      crun += c[k];
      // rows longer than 32: sorted by k_rows' extra blocks
      if (c[k] > 32) L.long_rows[atomicAdd(L.lcnt + 0, 1)] = base + t * kScanPer + k;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
      const int i = k * kBT + t;
      if (i < n) L.row_ptr[base + i] = buf[pad(i)];
    }
    if (last_tile && t == 0) L.row_ptr[len] = (int)(cpre + cagg);
    if (j == 0)
      for (int r = t; r <= L.R; r += kBT) L.o_rel_row_off[r] = L.key_base[r];
    return;
  }
  // slots: Y row numbering (presence prefix) and column starts (count prefix)
  {
    const int i0 = base + t * kScanPer;
    int r = 0;
    {
      int lo = 0, hi = L.R;                            // slot_base[lo] <= i0 < slot_base[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (L.slot_base[mid] <= i0) lo = mid; else hi = mid;
      }
      r = lo;
    }
#pragma unroll
    for (int k = 0; k < kScanPer; k++) {
      const int i = i0 + k;
      if (i < len && c[k] > 0) {
        while (r + 1 < L.R && L.slot_base[r + 1] <= i) r++;
        L.y_src[frun] = i - L.slot_base[r];
        if (L.csc) {
          L.col_ptr[frun] = (int)crun;
          // hub columns (> 32 entries): sorted by k_cols' extra blocks
          if (c[k] > 32) L.long_cols[atomicAdd(L.lcnt + 1, 1)] = (int)frun;
        }
      }
      // encoded: prefix if present, -1 - prefix if absent
      fbuf[pad(t * kScanPer + k)] = c[k] > 0 ? (int)frun : -1 - (int)frun;
      frun += c[k] > 0;
      crun += c[k];
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanPer; k++) {
    const int i = k * kBT + t;
    if (i < n) {
      const int f = fbuf[pad(i)];
      L.slot_y[base + i] = f >= 0 ? f : -1;
    }
  }
  // rel_y_off[r] = number of present slots before slot_base[r]
  for (int r = t; r <= L.R; r += kBT) {
    const int q = L.slot_base[r];
    if (q >= base && q < base + n) {
      const int f = fbuf[pad(q - base)];
      L.o_rel_y_off[r] = f >= 0 ? f : -1 - f;
    } else if (q >= len && last_tile) {
      L.o_rel_y_off[r] = (int)(fpre + fagg);
    }
  }
  if (last_tile && t == 0) {
    L.U_dev[0] = (int)(fpre + fagg);
    if (L.csc) L.col_ptr[fpre + fagg] = (int)(cpre + cagg);    // col_ptr[U] = valid edges
  }
}

// -------------------------------------------------------------- k_scatter --
__global__ void __launch_bounds__(kBT)
k_scatter(const __grid_constant__ BuildParams bp) {
  HF_PDL_ENTRY();
  int j;
  const BLayer& L = bp.lay[layer_of(bp.p, K_SCATTER, &j)];
  const int nvalid = L.row_ptr[L.rows];
  const int e0 = j * kEdgeTile;
  int key[kEPT], slot[kEPT], pos[kEPT], c[kEPT];
#pragma unroll
  for (int q = 0; q < kEPT; q++) {
    const int e = e0 + q * kBT + threadIdx.x;
    key[q] = e < L.N ? L.key_e[e] : -1;
    slot[q] = key[q] >= 0 ? L.slot_e[e] : 0;
  }
#pragma unroll
  for (int q = 0; q < kEPT; q++) {
    const int e = e0 + q * kBT + threadIdx.x;
    // one-run row: input order directly; else the arrival rank (k_rows sorts)
    const int rn = key[q] >= 0 ? L.runs[key[q]] : 0;
    const int f = rn == 1 ? L.first[key[q]] : 0;
    // several runs: an arrival ticket (k_rows sorts those rows)
    const int rk = (key[q] >= 0 && rn != 1) ? atomicAdd(L.rcur + key[q], 1) : 0;
    pos[q] = key[q] >= 0 ? L.row_ptr[key[q]] + (rn == 1 ? e - f : rk) : 0;
    c[q] = key[q] >= 0 ? (L.ynum ? L.slot_y[slot[q]] : (L.xg ? L.xg[slot[q]] : slot[q])) : 0;
  }
#pragma unroll
  for (int q = 0; q < kEPT; q++) {
    const int e = e0 + q * kBT + threadIdx.x;
    if (e < L.N && e >= nvalid) {      // tail positions [nvalid, N): one writer each
      L.eperm[e] = -1;
      L.col[e] = -1;
      if (L.csc) { L.csc_pos[e] = -1; L.csc_row[e] = -1; L.csc_col[e] = -1; }
    }
    if (key[q] < 0) continue;
    L.eperm[pos[q]] = e;
    L.col[pos[q]] = c[q];
  }
}

// ----------------------------------------------------------------- k_rows --
// Warp per 32 consecutive merged rows.  Their CSR span [row_ptr[r0],
// row_ptr[r0+32]) is contiguous: staged in shared memory, every row <= 32
// sorted by original column in registers (half warp per row <= 16, whole warp
// <= 32) and written back; the span is then placed into the CSC with its
// atomic slot requests batched (8 per lane in flight).  Rows longer than 32
// go to a block-local list, sorted and placed by the whole block at the end.
__device__ __forceinline__ void row_sorted(const BLayer& L, bool staged, int* sk, int* sv,
                                           int span_b, int b, int i, int key, int val) {
  L.eperm[b + i] = key;
  L.col[b + i] = val;
  if (staged) {
    sk[b - span_b + i] = key;
    sv[b - span_b + i] = val;
  }
}

__global__ void __launch_bounds__(kBT)
k_rows(const __grid_constant__ BuildParams bp) {
  HF_PDL_ENTRY();
  extern __shared__ __align__(16) int sm[];
  int j;
  const BLayer& L = bp.lay[layer_of(bp.p, K_ROWS, &j)];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (j >= L.rows_reg) {
    // rows longer than 32 (listed by k_scan; not produced by fanout <= 32
    // sampling): one block per row
    const int nl = L.lcnt[0];
    for (int k = j - L.rows_reg; k < nl; k += kLongRowBlocks) {
      const int row = L.long_rows[k];
      const int b = L.row_ptr[row], e = L.row_ptr[row + 1];
      block_sort_segment<kBlockRankR>(L.eperm, L.col, b, e, sm, L.gk, L.gv);
      if (L.csc)
        for (int p = b + threadIdx.x; p < e; p += kBT) place_entry(L, row, p, L.col[p]);
      __syncthreads();
    }
    return;
  }
  const int r0 = (j * kNW + w) * kRowsW;
  if (r0 < L.rows) {
    const int nr = min(kRowsW, L.rows - r0);
    int* sk = sm + w * 2 * kSpanR;
    int* sv = sk + kSpanR;
    const int rb = L.row_ptr[r0 + min(lane, nr)];                 // start of row r0+lane
    const int re = L.row_ptr[r0 + min(lane + 1, nr)];             // its end
    const int n = lane < nr ? re - rb : 0;
    // rows made of several input runs need the sort (one-run rows are in
    // input order already, k_scatter)
    const bool multi = n > 1 && L.runs[r0 + lane] > 1;
    const unsigned need = __ballot_sync(0xffffffffu, multi);
    if (!need && !L.csc) return;
    const int span_b = __shfl_sync(0xffffffffu, rb, 0);
    const int span_e = __shfl_sync(0xffffffffu, re, nr - 1);
    const int span = span_e - span_b;
    const bool staged = span <= kSpanR;
    if (staged) {
      stage2(L.eperm + span_b, L.col + span_b, span, span, sk, sv, lane, 32);
      __syncwarp();
    }
    // rows of <= 16 entries: two per iteration (one per half warp)
    const int hl = lane & 15, half = lane >> 4;
    for (int q = 0; q < nr; q += 2) {
      const int row = q + half;
      const int src = row < nr ? row : 0;
      const int b = __shfl_sync(0xffffffffu, rb, src);
      const int nn = __shfl_sync(0xffffffffu, n, src);
      const bool mine = row < nr && nn <= 16 && ((need >> src) & 1u);
      int key = 0x7fffffff, val = 0;
      if (mine && hl < nn) {
        key = staged ? sk[b - span_b + hl] : L.eperm[b + hl];
        val = staged ? sv[b - span_b + hl] : L.col[b + hl];
      }
      if (__any_sync(0xffffffffu, mine && nn > 1)) half_sort_regs(key, val, hl);
      __syncwarp();
      if (mine && hl < nn) row_sorted(L, staged, sk, sv, span_b, b, hl, key, val);
    }
    // rows of 17..32 entries: whole warp, one after another
    unsigned mid = __ballot_sync(0xffffffffu, lane < nr && n > 16 && n <= 32) & need;
    while (mid) {
      const int src = __ffs(mid) - 1;
      mid &= mid - 1;
      const int b = __shfl_sync(0xffffffffu, rb, src), nn = __shfl_sync(0xffffffffu, n, src);
      int key = 0x7fffffff, val = 0;
      if (lane < nn) {
        key = staged ? sk[b - span_b + lane] : L.eperm[b + lane];
        val = staged ? sv[b - span_b + lane] : L.col[b + lane];
      }
      warp_sort_regs(key, val, lane);
      __syncwarp();
      if (lane < nn) row_sorted(L, staged, sk, sv, span_b, b, lane, key, val);
    }
    __syncwarp();
    if (L.csc) {
      // CSC placement of the span's rows of <= 32 entries
      constexpr int kB = 8;
      for (int i0 = 0; i0 < span; i0 += 32 * kB) {
        int c[kB], row[kB], ws[kB], cp[kB];
#pragma unroll
        for (int k = 0; k < kB; k++) {
          const int i = i0 + k * 32 + lane;
          const int ic = min(i, span - 1);
          // row of entry ic: the last row of the group whose start is <= ic
          // (an empty row shares its start with the next row, which is later)
          int lo = 0;
#pragma unroll
          for (int stp = 16; stp; stp >>= 1) {
            const int cand = lo + stp;
            const int bs = __shfl_sync(0xffffffffu, rb, cand < nr ? cand : 0);
            if (cand < nr && bs - span_b <= ic) lo = cand;
          }
          const int nlo = __shfl_sync(0xffffffffu, n, lo);
          row[k] = lo;
          c[k] = (i < span && nlo <= 32) ? (staged ? sv[i] : L.col[span_b + i]) : -1;
        }
        // slot requests: warp-aggregated (a hub source appears in many of the
        // warp's 32 rows), all of the batch in flight together
        unsigned pc[kB];
#pragma unroll
        for (int k = 0; k < kB; k++) pc[k] = __match_any_sync(0xffffffffu, c[k] >= 0 ? c[k] : -1 - lane);
#pragma unroll
        for (int k = 0; k < kB; k++) {
          const bool lead = c[k] >= 0 && lane == __ffs(pc[k]) - 1;
          ws[k] = lead ? atomicAdd(L.ccur + c[k], __popc(pc[k])) : 0;
          cp[k] = c[k] >= 0 ? L.col_ptr[c[k]] : 0;
        }
#pragma unroll
        for (int k = 0; k < kB; k++)
          ws[k] = __shfl_sync(0xffffffffu, ws[k], __ffs(pc[k]) - 1) +
                  __popc(pc[k] & ((1u << lane) - 1u));
#pragma unroll
        for (int k = 0; k < kB; k++)
          if (c[k] >= 0) {
            const int w2 = cp[k] + ws[k];
            L.csc_pos[w2] = span_b + i0 + k * 32 + lane;
            L.csc_row[w2] = r0 + row[k];
            L.csc_col[w2] = c[k];
          }
      }
    }
  }
}

// ----------------------------------------------------------------- k_cols --
// Warp per 32 consecutive CSC columns (Y rows < U): lane per column for
// <= 16 entries (insertion sort in shared memory), whole warp for 17..32;
// longer (hub) columns: warp rank sort in shared memory for <= kWarpRank,
// block rank sort beyond.  Blocks past U write the col_ptr tail (= valid
// edges).
__global__ void __launch_bounds__(kBT)
k_cols(const __grid_constant__ BuildParams bp) {
  HF_PDL_ENTRY();
  extern __shared__ __align__(16) int sm[];
  constexpr int kThreadCap = 16;
  int j;
  const BLayer& L = bp.lay[layer_of(bp.p, K_COLS, &j)];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (j >= L.cols_reg) {
    // hub columns (> 32 entries, listed by k_scan), spread over the extra
    // blocks: <= kWarpRank entries by one warp (rank sort), longer by the
    // whole block (bitonic)
    const int xb = j - L.cols_reg;
    const int n_extra = L.cols_xtra;
    const int nl = L.lcnt[1];
    {
      int* sk = sm + w * 2 * kWarpRank;
      int* sv = sk + kWarpRank;
      for (int k = xb * kNW + w; k < nl; k += n_extra * kNW) {
        const int u = L.long_cols[k];
        const int b = L.col_ptr[u], e = L.col_ptr[u + 1], n = e - b;
        if (n > kWarpRank) continue;
        stage2(L.csc_pos + b, L.csc_row + b, n, (n + 3) & ~3, sk, sv, lane, 32);
        __syncwarp();
        rank_scatter<kWarpRank / 32>(sk, sv, n, lane, 32, L.csc_pos + b, L.csc_row + b);
        __syncwarp();
      }
    }
    __syncthreads();
    for (int k = xb; k < nl; k += n_extra) {
      const int u = L.long_cols[k];
      const int b = L.col_ptr[u], e = L.col_ptr[u + 1];
      if (e - b <= kWarpRank) continue;
      block_sort_segment<kBlockRank>(L.csc_pos, L.csc_row, b, e, sm, L.gk, L.gv);
    }
    return;
  }
  const int U = *L.U_dev;
  if ((j + 1) * kSegTile > U) {                   // col_ptr tail (U, U_max] of this tile
    const int nvalid = L.row_ptr[L.rows];
    const int hi = min((j + 1) * kSegTile - 1, L.U_max);
    for (int u = max(j * kSegTile, U + 1) + threadIdx.x; u <= hi; u += kBT) L.col_ptr[u] = nvalid;
    if (j * kSegTile >= U) return;
  }
  const int u0 = (j * kNW + w) * kSegRows;
  if (u0 < U) {
    const int nu = min(kSegRows, U - u0);
    int* sk = sm + w * 2 * kSpan;
    int* sv = sk + kSpan;
    const int cb = L.col_ptr[u0 + min(lane, nu)];
    const int ce = L.col_ptr[u0 + min(lane + 1, nu)];
    const int n = lane < nu ? ce - cb : 0;
    const int span_b = __shfl_sync(0xffffffffu, cb, 0);
    const int span_e = __shfl_sync(0xffffffffu, ce, nu - 1);
    const int span = span_e - span_b;
    // stage the span unless hub columns make it long (then read from global)
    const bool staged = span <= kSpan;
    if (staged) {
      stage2(L.csc_pos + span_b, L.csc_row + span_b, span, span, sk, sv, lane, 32);
      __syncwarp();
    }
    if (n > 1 && n <= kThreadCap) {
      // insertion sort of the lane's column in shared memory (columns hold
      // ~2 entries on average: a fixed 16-element network wasted most work).
      // Unstaged span: the lane copies its column to a private 16-slot area.
      int* ks = staged ? sk + (cb - span_b) : sk + lane * kThreadCap;
      int* vs = staged ? sv + (cb - span_b) : sv + lane * kThreadCap;
      if (!staged)
        for (int i = 0; i < n; i++) {
          ks[i] = L.csc_pos[cb + i];
          vs[i] = L.csc_row[cb + i];
        }
      for (int i = 1; i < n; i++) {
        const int k0 = ks[i], v0 = vs[i];
        int q = i - 1;
        while (q >= 0 && ks[q] > k0) {
          ks[q + 1] = ks[q];
          vs[q + 1] = vs[q];
          q--;
        }
        ks[q + 1] = k0;
        vs[q + 1] = v0;
      }
      for (int i = 0; i < n; i++) {
        L.csc_pos[cb + i] = ks[i];
        L.csc_row[cb + i] = vs[i];
      }
    }
    __syncwarp();
    unsigned mid = __ballot_sync(0xffffffffu, n > kThreadCap && n <= 32);
    while (mid) {
      const int src = __ffs(mid) - 1;
      mid &= mid - 1;
      const int b = __shfl_sync(0xffffffffu, cb, src), nn = __shfl_sync(0xffffffffu, n, src);
      int key = 0x7fffffff, val = 0;
      if (lane < nn) {
        key = staged ? sk[b - span_b + lane] : L.csc_pos[b + lane];
        val = staged ? sv[b - span_b + lane] : L.csc_row[b + lane];
      }
      warp_sort_regs(key, val, lane);
      if (lane < nn) {
        L.csc_pos[b + lane] = key;
        L.csc_row[b + lane] = val;
      }
    }
  }
}

// ------------------------------------------------------------- host side --
long long umax_of(const LayerMeta& m) { return m.N < m.S ? m.N : m.S; }
int tiles(long long n, long long per) { return (int)std::max<long long>(1, (n + per - 1) / per); }

// Per-layer workspace: zero zone (cnt [rows + S], ccur [U_max + 1], scan tile
// statuses) and scratch.  The zero zones of all layers of a call are laid
// out first and contiguously (one memset), the scratch after them.
struct LayerWs {
  long long zero_bytes, scratch_bytes;
};

LayerWs layer_ws_sizes(const LayerMeta& m, bool csc) {
  const long long U_max = umax_of(m);
  LayerWs s;
  s.zero_bytes = carve_bytes((long long)m.rows + m.S, 4) + 2 * carve_bytes(m.rows, 4) +
                 (csc ? carve_bytes(U_max + 1, 4) : 0) + carve_bytes(2, 4) +
                 carve_bytes(2ll * (tiles(m.rows, kScanTile) + tiles(m.S, kScanTile)), 4);
  s.scratch_bytes = carve_bytes(m.N, 4) * 4 +              // key_e slot_e gk gv
                    carve_bytes(m.rows, 4) + carve_bytes(U_max, 4) +  // long lists
                    carve_bytes(m.rows, 4);                           // first
  return s;
}

void carve_layer(const LayerMeta& m, bool csc, char*& zp, char*& sp, BLayer* L) {
  const long long U_max = umax_of(m);
  L->t_rows = tiles(m.rows, kScanTile);
  L->t_slots = tiles(m.S, kScanTile);
  L->cnt = carve<int>(zp, (long long)m.rows + m.S);
  L->runs = carve<int>(zp, m.rows);
  L->rcur = carve<int>(zp, m.rows);
  L->ccur = csc ? carve<int>(zp, U_max + 1) : nullptr;
  L->lcnt = carve<int>(zp, 2);
  L->sst = reinterpret_cast<unsigned long long*>(
      carve<int>(zp, 2ll * (L->t_rows + L->t_slots)));
  L->key_e = carve<int>(sp, m.N);
  L->slot_e = carve<int>(sp, m.N);
  L->gk = carve<int>(sp, m.N);
  L->gv = carve<int>(sp, m.N);
  L->long_rows = carve<int>(sp, m.rows);
  L->long_cols = carve<int>(sp, U_max);
  L->first = carve<int>(sp, m.rows);
}

}  // namespace
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
  if (ws_bytes) {
    const LayerWs w = layer_ws_sizes(m, true);
    *ws_bytes = (size_t)(w.zero_bytes + w.scratch_bytes);
  }
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
  std::vector<LayerMeta> metas(num_layers);
  for (int l = 0; l < num_layers; l++) {
    hifuse_status rc = make_meta(&shapes[l], &metas[l]);
    if (rc != HIFUSE_OK) return rc;
    const LayerMeta& m = metas[l];
    const hifuse_csr& o = out[l];
    // y_src == NULL: X-row mode (col = the source's row in the layer's X, no
    // Y numbering, no CSC; rel_y_off / U_dev / slot_y unused)
    const bool ynum = o.y_src != nullptr;
    if (!o.rel_row_off || !o.row_ptr || (ynum && (!o.rel_y_off || !o.U_dev)) ||
        (m.N > 0 && (!d_src_local[l] || !d_dst_local[l] || !d_edge_id[l] || !o.col ||
                     !o.eperm)) ||
        (!o.col_ptr != !o.csc_pos || !o.col_ptr != !o.csc_row || !o.col_ptr != !o.csc_col) ||
        (ynum && m.S > 0 && !o.slot_y) || (!ynum && o.col_ptr))
      return HIFUSE_ERR_INVALID_ARG;
    if (m.N >= (1 << 30) || m.S >= (1 << 30)) return HIFUSE_ERR_UNSUPPORTED;   // status packing
  }
  // the layer sets of kMaxL layers run in order, each from the start of d_ws
  size_t need = 0;
  for (int l0 = 0; l0 < num_layers; l0 += kMaxL) {
    size_t set = 0;
    for (int l = l0; l < std::min(num_layers, l0 + kMaxL); l++) {
      const LayerWs w = layer_ws_sizes(metas[l], out[l].col_ptr != nullptr);
      set += w.zero_bytes + w.scratch_bytes;
    }
    need = std::max(need, set);
  }
  if (!d_ws || need > ws_bytes) return HIFUSE_ERR_WORKSPACE;
  set_max_smem((const void*)k_scan, (int)kSmemScan);
  set_max_smem((const void*)k_rows, (int)kSmemRows);
  set_max_smem((const void*)k_cols, (int)kSmem);
  for (int l0 = 0; l0 < num_layers; l0 += kMaxL) {
    const int nl = std::min(kMaxL, num_layers - l0);
    BuildParams bp;
    memset(&bp, 0, sizeof(bp));
    BPlan& P = bp.p;
    P.L = nl;
    P.E = num_graph_edges;
    P.edge_type = d_edge_type;
    P.rel_off = (const long long*)d_rel_edge_off;
    P.status = d_status;
    long long zero_total = 0;
    for (int q = 0; q < nl; q++)
      zero_total += layer_ws_sizes(metas[l0 + q], out[l0 + q].col_ptr != nullptr).zero_bytes;
    char* zp = (char*)d_ws;
    char* sp = (char*)d_ws + zero_total;
    int blocks[kKerns][kMaxL] = {};
    for (int q = 0; q < nl; q++) {
      const LayerMeta& m = metas[l0 + q];
      const hifuse_csr& o = out[l0 + q];
      BLayer& L = bp.lay[q];
      const bool csc = o.col_ptr != nullptr;
      carve_layer(m, csc, zp, sp, &L);
      L.ynum = o.y_src != nullptr;
      if (!L.ynum) L.t_slots = 0;                  // no slot segment to scan
      L.R = m.R; L.N = m.N; L.rows = m.rows; L.S = m.S;
      L.U_max = (int)umax_of(m);
      L.csc = csc;
      for (int r = 0; r <= m.R; r++) {
        L.key_base[r] = m.rel_row_off[r];
        L.slot_base[r] = m.slot_off[r];
      }
      for (int r = 0; r < m.R; r++) {
        L.src_lim[r] = m.n_src[m.rel_src[r]];
        L.dst_lim[r] = m.n_dst[m.rel_dst[r]];
        L.xoff[r] = m.type_src_off[m.rel_src[r]];
      }
      L.src = d_src_local[l0 + q];
      L.dst = d_dst_local[l0 + q];
      L.eid = (const long long*)d_edge_id[l0 + q];
      L.o_rel_row_off = o.rel_row_off; L.row_ptr = o.row_ptr; L.col = o.col; L.eperm = o.eperm;
      L.o_rel_y_off = o.rel_y_off; L.y_src = o.y_src; L.col_ptr = o.col_ptr;
      L.csc_pos = o.csc_pos; L.csc_row = o.csc_row; L.csc_col = o.csc_col; L.slot_y = o.slot_y; L.U_dev = o.U_dev;
      L.xg = L.ynum ? nullptr : o.x_gather;
      const int et = m.N > 0 ? tiles(m.N, kEdgeTile) : 0;
      blocks[K_CLASSIFY][q] = et;
      blocks[K_SCAN][q] = L.t_rows + L.t_slots;
      blocks[K_SCATTER][q] = et;
      L.rows_reg = m.rows > 0 ? tiles(m.rows, kRowsTile) : 0;
      L.cols_reg = csc ? tiles((long long)L.U_max + 1, kSegTile) : 0;
      L.cols_xtra = csc && m.N > 0 ? 2 * sm_count() : 0;
      blocks[K_ROWS][q] = L.rows_reg + (m.rows > 0 ? kLongRowBlocks : 0);
      blocks[K_COLS][q] = L.cols_reg + L.cols_xtra;
    }
    int total[kKerns];
    for (int k = 0; k < kKerns; k++) {
      int acc = 0;
      for (int q = 0; q <= kMaxL; q++) {
        P.blk_off[k][q] = acc;
        if (q < nl) acc += blocks[k][q];
      }
      total[k] = acc;
    }
    cudaMemsetAsync(d_ws, 0, (size_t)zero_total, s);
    HF_LAUNCH(k_classify, total[K_CLASSIFY], kBT, 0, s, bp);
    HF_LAUNCH(k_scan, total[K_SCAN], kBT, kSmemScan, s, bp);
    HF_LAUNCH(k_scatter, total[K_SCATTER], kBT, 0, s, bp);
    HF_LAUNCH(k_rows, total[K_ROWS], kBT, kSmemRows, s, bp);
    HF_LAUNCH(k_cols, total[K_COLS], kBT, kSmem, s, bp);
  }
  return last_cuda();
}

}  // extern "C"

// ------------------------------------------------- edge-type preprocessing --
namespace hf {
namespace {
// d_rel_edge_off[r] = lower bound of r in the (sorted) edge-type table.
__global__ void k_et_offsets(const int* __restrict__ et, long long E, int R,
                             long long* __restrict__ off) {
  HF_PDL_ENTRY();
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
  HF_PDL_ENTRY();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E) return;
  const int v = et[i];
  if (v < 0 || v >= R || (i > 0 && et[i - 1] > v)) atomicOr(status, HIFUSE_ST_UNSORTED_TYPES);
}
}  // namespace
}  // namespace hf

extern "C" hifuse_status hifuse_edge_type_offsets(const int32_t* d_edge_type,
                                                  int64_t num_graph_edges, int num_rels,
                                                  int64_t* d_rel_edge_off, int32_t* d_status,
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

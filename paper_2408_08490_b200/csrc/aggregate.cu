// aggregate.cu -- A4 (merged neighbour aggregation, Alg. 1 lines
// 246-268) and A6b (its transpose, the aggregation backward).
//
// Merging (Alg. 1) concatenates every semantic graph's gathered
// source features and destination indices so that ONE Aggregate call serves
// all relations.  Here the concatenation is virtual: the build's segmented
// CSR indexes the merged projected matrix Y directly, so FeatureCat is never
// materialised and A4 is a single relation-agnostic CSR gather-reduce.
//
// Mapping (B200): one warp per merged (relation, destination) row; a row of D
// fp32 is D/4 float4 lanes, so D = 128 uses the whole warp on one edge and
// D = 64 runs two half-warp edge streams that merge at the end.  Up to 32
// column indices are fetched with one coalesced load and broadcast with
// shuffles; the gathers of UNROLL edges per stream are issued back to back to
// keep several 256-512 B row loads in flight per warp (HBM latency hiding).
#include <cuda_bf16.h>
#include <cstring>
#include "common.cuh"

namespace hf {

static constexpr int kWarpsPerBlock = 8;
static constexpr int kUnroll = 4;
// gathers in flight per stream for the raw-feature (evict-first) aggregation
#ifndef HF_FEAT_UNROLL
#define HF_FEAT_UNROLL 4
#endif
static constexpr int kFeatUnroll = HF_FEAT_UNROLL;
// feature aggregations of at most kLatRows merged rows (under one wave of
// warps: latency- not bandwidth-bound, e.g. the inner layer) use the latency
// variant of agg_row: kLatUnroll loads in flight, predicated tail
#ifndef HF_LAT_ROWS
#define HF_LAT_ROWS 8192
#endif
#ifndef HF_LAT_UNROLL
#define HF_LAT_UNROLL 8
#endif
static constexpr long long kLatRows = HF_LAT_ROWS;
static constexpr int kLatUnroll = HF_LAT_UNROLL;

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 f4fma(float s, float4 y, float4 a) {
  return make_float4(fmaf(s, y.x, a.x), fmaf(s, y.y, a.y), fmaf(s, y.z, a.z), fmaf(s, y.w, a.w));
}
__device__ __forceinline__ float4 f4shfl_xor(float4 v, int o) {
  return make_float4(__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o),
                     __shfl_xor_sync(0xffffffffu, v.z, o), __shfl_xor_sync(0xffffffffu, v.w, o));
}
// y + s * a elementwise as fmaf(s, a, y): the score-chain term of dYt
// (k_dy_score's arithmetic, bit for bit)
__device__ __forceinline__ float4 f4fma_into(float s, float4 a, float4 y) {
  return make_float4(fmaf(s, a.x, y.x), fmaf(s, a.y, y.y), fmaf(s, a.z, y.z), fmaf(s, a.w, y.w));
}
__device__ __forceinline__ float leaky(float x, float slope) { return x > 0.f ? x : slope * x; }
// Attention logit of an edge from its source score ss and destination score
// sd: additive GAT (reading C6) LeakyReLU(ss + sd), or multiplicative (MUL,
// reading C23: one query / key unit per head) ss * sd; and its partials.
template <bool MUL>
__device__ __forceinline__ float att_logit(float ss, float sd, float slope) {
  return MUL ? __fmul_rn(ss, sd) : leaky(ss + sd, slope);   // rounded product: no fma contraction
}
template <bool MUL>
__device__ __forceinline__ float dlogit_dss(float ss, float sd, float slope) {
  return MUL ? sd : ((ss + sd) > 0.f ? 1.f : slope);
}
template <bool MUL>
__device__ __forceinline__ float dlogit_dsd(float ss, float sd, float slope) {
  return MUL ? ss : ((ss + sd) > 0.f ? 1.f : slope);
}
__device__ __forceinline__ float4 ldg4(const float4* p) { return __ldg(p); }
// Raw feature rows of the aggregate-first input layer: read once per batch
// (the batch's distinct rows roughly fill the L2), so they are loaded with
// the evict-first (streaming) policy and do not push the layer's reused
// lines (row pointers, column ids, the output) out of the L2.
__device__ __forceinline__ float4 ldcs4(const float4* p) { return __ldcs(p); }

// ------------------------------------------------------------ forward SUM/MEAN
// One merged row (warp; D = 64: two edge streams of 16 lanes): the row's sum
// (mean: divided by its degree), in every stream-0 lane's float4 slice.
// UNR > 0 (latency variant, small layers): UNR loads in flight and the tail
// as one predicated batch (masked slots add +0) instead of one dependent load
// per remaining edge -- same add order.
template <int D, bool MEAN, bool CS, int UNR = 0>
__device__ __forceinline__ float4 agg_row(long long row, const int* __restrict__ row_ptr,
                                          const int* __restrict__ col,
                                          const float4* __restrict__ Y, int lane) {
  constexpr int LPR = D / 4;              // lanes per row stream
  constexpr int NS = 32 / LPR;            // edge streams per warp
  const int sl = lane % LPR, sid = lane / LPR;
  const int b = row_ptr[row], e = row_ptr[row + 1];
  constexpr int UN = UNR ? UNR : (CS ? kFeatUnroll : kUnroll);   // (same add order at any unroll)
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int base = b; base < e; base += 32) {
    const int n = min(32, e - base);
    const int my_col = lane < n ? __ldg(col + base + lane) : 0;
    int k = 0;
    for (; k + NS * UN <= n; k += NS * UN) {
      float4 v[UN];
#pragma unroll
      for (int u = 0; u < UN; u++) {
        int c = __shfl_sync(0xffffffffu, my_col, k + u * NS + sid);
        v[u] = CS ? ldcs4(Y + (long long)c * LPR + sl) : ldg4(Y + (long long)c * LPR + sl);
      }
#pragma unroll
      for (int u = 0; u < UN; u++) acc = f4add(acc, v[u]);
    }
    if (UNR > 0) {
      if (k < n) {
        float4 v[UN];
#pragma unroll
        for (int u = 0; u < UN; u++) {
          const int idx = k + u * NS + sid;
          const int c = __shfl_sync(0xffffffffu, my_col, idx < n ? idx : 0);
          v[u] = idx < n ? (CS ? ldcs4(Y + (long long)c * LPR + sl) : ldg4(Y + (long long)c * LPR + sl))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < UN; u++) acc = f4add(acc, v[u]);
      }
    } else {
      for (; k < n; k += NS) {
        int idx = k + sid;
        int c = __shfl_sync(0xffffffffu, my_col, idx < n ? idx : 0);
        if (idx < n)
          acc = f4add(acc, CS ? ldcs4(Y + (long long)c * LPR + sl) : ldg4(Y + (long long)c * LPR + sl));
      }
    }
  }
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) acc = f4add(acc, f4shfl_xor(acc, o));
  if (MEAN && e > b) {
    float dg = (float)(e - b);
    acc = make_float4(__fdiv_rn(acc.x, dg), __fdiv_rn(acc.y, dg), __fdiv_rn(acc.z, dg),
                      __fdiv_rn(acc.w, dg));
  }
  return acc;
}

template <int D, bool MEAN, bool CS = false, int UNR = 0>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_fwd(long long rows, const int* __restrict__ row_ptr, const int* __restrict__ col,
          const float4* __restrict__ Y, float4* __restrict__ Z) {
  HF_PDL_ENTRY();
  constexpr int LPR = D / 4;
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (row >= rows) return;
  const float4 acc = agg_row<D, MEAN, CS, UNR>(row, row_ptr, col, Y, lane);
  if (lane < LPR) Z[row * LPR + lane] = acc;
}

// A5 fused into A4 (hifuse_aggregate_fuse_fwd): the warp that completes the
// LAST relation row (r, i) of destination (t, i) -- a per-destination arrival
// counter, fenced -- forms H_t[i] = act(R0 + b + sum_r Z[(r, i)]) in
// hifuse_semantic_fuse's order (relations in relation order, reading the
// other rows' Z from L2) and resets the counter (graph-safe).  Destinations of
// a type no relation enters (no rows) get H = act(R0 + b) from the blocks past
// the aggregation grid.  Removes the fusion launch and its Z re-read pass.
struct FuseEpi {
  int R, relu;
  unsigned agg_blocks;                 // blocks of the aggregation part
  int n_orph;                          // destination rows of types without relations
  int rel_row_off[HF_MAX_R + 1];
  int rel_dst[HF_MAX_R];
  int type_dst_off[HF_MAX_T + 1];
  int list_off[HF_MAX_T + 1];          // relations into type t: rel_rows[list_off[t] ..)
  int rel_rows[HF_MAX_R];
  int n_orph_types;
  int orph_t[HF_MAX_T];                // orphan types and their row prefix
  int orph_off[HF_MAX_T + 1];
};

template <int D>
__device__ __forceinline__ void fuse_dst(const FuseEpi& f, int t, int i, int lane,
                                         const float4* __restrict__ Z,
                                         const float4* __restrict__ R0,
                                         const float4* __restrict__ bias,
                                         float4* __restrict__ H) {
  constexpr int LPR = D / 4;
  if (lane >= LPR) return;
  const long long o = f.type_dst_off[t] + i;
  float4 v = R0 ? __ldcg(R0 + o * LPR + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
  if (bias) {
    const float4 b = bias[t * LPR + lane];
    v.x += b.x; v.y += b.y; v.z += b.z; v.w += b.w;
  }
  for (int k = f.list_off[t]; k < f.list_off[t + 1]; k++) {
    const float4 z = __ldcg(Z + (long long)(f.rel_rows[k] + i) * LPR + lane);
    v.x += z.x; v.y += z.y; v.z += z.z; v.w += z.w;
  }
  if (f.relu) {
    v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
  }
  H[o * LPR + lane] = v;
}

template <int D, bool MEAN>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_fuse_fwd(long long rows, const int* __restrict__ row_ptr, const int* __restrict__ col,
               const float4* __restrict__ Y, float4* __restrict__ Z, const FuseEpi f,
               const float4* __restrict__ R0, const float4* __restrict__ bias,
               float4* __restrict__ H, int* __restrict__ cnt) {
  HF_PDL_ENTRY();
  constexpr int LPR = D / 4;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x >= f.agg_blocks) {                 // destinations without relation rows
    const int q = (blockIdx.x - f.agg_blocks) * kWarpsPerBlock + (threadIdx.x >> 5);
    if (q >= f.n_orph) return;
    int a = 0;
    while (a + 1 < f.n_orph_types && f.orph_off[a + 1] <= q) a++;
    fuse_dst<D>(f, f.orph_t[a], q - f.orph_off[a], lane, Z, R0, bias, H);
    return;
  }
  const long long row = (long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (row >= rows) return;
  const float4 acc = agg_row<D, MEAN, false>(row, row_ptr, col, Y, lane);
  if (lane < LPR) Z[row * LPR + lane] = acc;
  const int r = upper_bound_i(f.rel_row_off, f.R + 1, (int)row) - 1;
  const int t = f.rel_dst[r], i = (int)row - f.rel_row_off[r];
  const int o = f.type_dst_off[t] + i;
  __threadfence();                                  // publish this Z row
  __syncwarp();
  int last = 0;
  if (lane == 0) last = atomicAdd(cnt + o, 1) == f.list_off[t + 1] - f.list_off[t] - 1;
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();                                  // the other rows' Z are visible
  if (lane == 0) cnt[o] = 0;                        // ready for the next call
  fuse_dst<D>(f, t, i, lane, Z, R0, bias, H);
}


// NEXT(3) byte diet: the aggregate-first input layer over a BF16 feature
// store (2 bytes per feature instead of 4 on the layer's dominant read).
// Rows are accumulated in fp32 in the same order as k_agg_fwd (the oracle is
// fed the BF16-rounded features).  A lane loads 16 B = 8 bf16;
// K = 128: 16 lanes per row, 2 edge streams per warp.  Blocks past the
// aggregation grid convert the layer's destination rows (the root term's X
// rows) to fp32 into Xdst[type_src_off[t] + i] for the tcgen05 GEMMs.
__device__ __forceinline__ void bf16x8_add(const uint4 q, float* a) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const float2 f = __bfloat1622float2(h[j]);
    a[2 * j] += f.x;
    a[2 * j + 1] += f.y;
  }
}

struct DstConv {
  int T;
  int n_dst[HF_MAX_T];
  int type_src_off[HF_MAX_T + 1];
  int dst_off[HF_MAX_T + 1];      // prefix over types of n_dst
};

// CS: evict-first loads of the gathered rows (raw feature-store rows, read
// once per batch); the BF16-Y path (rows reused by several edges) keeps them.
template <int D, bool MEAN, bool CS = false>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_fwd_bf16(long long rows, unsigned agg_blocks, const int* __restrict__ row_ptr,
               const int* __restrict__ col, const uint4* __restrict__ Xb,
               float4* __restrict__ Z, DstConv dc, const int* __restrict__ gather_ids,
               float4* __restrict__ Xdst) {
  HF_PDL_ENTRY();
  constexpr int LPR = D / 8;              // lanes per row stream (8 bf16 each)
  constexpr int NS = 32 / LPR;            // edge streams per warp
  const int lane = threadIdx.x & 31;
  if (blockIdx.x >= agg_blocks) {
    // destination rows -> fp32 (one thread per 8 features)
    const long long i = (long long)(blockIdx.x - agg_blocks) * blockDim.x + threadIdx.x;
    if (!Xdst || i >= (long long)dc.dst_off[dc.T] * LPR) return;
    const int o = (int)(i / LPR), c8 = (int)(i % LPR);
    const int t = upper_bound_i(dc.dst_off, dc.T + 1, o) - 1;
    const int x = dc.type_src_off[t] + (o - dc.dst_off[t]);
    const long long g = gather_ids ? (long long)gather_ids[x] : (long long)x;
    const uint4 q = __ldg(Xb + g * LPR + c8);
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    bf16x8_add(q, a);
    Xdst[(long long)x * (D / 4) + 2 * c8] = make_float4(a[0], a[1], a[2], a[3]);
    Xdst[(long long)x * (D / 4) + 2 * c8 + 1] = make_float4(a[4], a[5], a[6], a[7]);
    return;
  }
  const int sl = lane % LPR, sid = lane / LPR;
  long long row = (long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int b = row_ptr[row], e = row_ptr[row + 1];
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int base = b; base < e; base += 32) {
    const int n = min(32, e - base);
    const int my_col = lane < n ? __ldg(col + base + lane) : 0;
    int k = 0;
    for (; k + NS * kUnroll <= n; k += NS * kUnroll) {
      uint4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        const int c = __shfl_sync(0xffffffffu, my_col, k + u * NS + sid);
        v[u] = CS ? __ldcs(Xb + (long long)c * LPR + sl) : __ldg(Xb + (long long)c * LPR + sl);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; u++) bf16x8_add(v[u], acc);
    }
    for (; k < n; k += NS) {
      const int idx = k + sid;
      const int c = __shfl_sync(0xffffffffu, my_col, idx < n ? idx : 0);
      if (idx < n)
        bf16x8_add(CS ? __ldcs(Xb + (long long)c * LPR + sl) : __ldg(Xb + (long long)c * LPR + sl), acc);
    }
  }
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
  if (sid == 0) {
    if (MEAN && e > b) {
      const float dg = (float)(e - b);
#pragma unroll
      for (int j = 0; j < 8; j++) acc[j] = __fdiv_rn(acc[j], dg);
    }
    Z[row * (D / 4) + 2 * sl] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    Z[row * (D / 4) + 2 * sl + 1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// Aggregate-first input layer: CSR position p -> the global feature row of its
// source, x = gather_ids[type_src_off[s(r)] + y_src[col[p]]] (r = relation of
// the compact Y id col[p]), so A4's kernel can gather raw features.
struct RelOff { int v[HF_MAX_R]; };   // type_src_off[s(r)] per relation

__global__ void __launch_bounds__(256)
k_col_to_x(int N, int R, const int* __restrict__ rel_y_off, RelOff so,
           const int* __restrict__ col, const int* __restrict__ y_src,
           const int* __restrict__ gather_ids, int* __restrict__ col_x) {
  HF_PDL_ENTRY();
  __shared__ int s_yo[HF_MAX_R + 1];
  __shared__ int s_so[HF_MAX_R];
  for (int i = threadIdx.x; i <= R; i += blockDim.x) {
    s_yo[i] = rel_y_off[i];
    if (i < R) s_so[i] = so.v[i];
  }
  __syncthreads();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int c = col[p];
  if (c < 0) { col_x[p] = 0; return; }       // tail past the valid edges: never read
  const int r = upper_bound_i(s_yo, R + 1, c) - 1;
  const int x = s_so[r] + y_src[c];
  col_x[p] = gather_ids ? gather_ids[x] : x;
}

// X-row build: col_x[p] = gather_ids[col[p]] (or col[p]); tail (-1) -> 0.
__global__ void __launch_bounds__(256)
k_xrow_to_feat(int N, const int* __restrict__ col, const int* __restrict__ gather_ids,
               int* __restrict__ col_x) {
  HF_PDL_ENTRY();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const int c = col[p];
  col_x[p] = c < 0 ? 0 : (gather_ids ? gather_ids[c] : c);
}

// ------------------------------------------------------------- forward GAT
// Per head h: two passes over the row's edges (rows are short): the max of the
// logits, then p = exp(l - max), sum p and sum p * Y.  stats = (max, sum p).
template <int D, bool MUL>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_fwd_gat(long long rows, int H, float slope, const int* __restrict__ row_ptr,
              const int* __restrict__ col, const float4* __restrict__ Y,
              const float* __restrict__ s_src, const float* __restrict__ s_dst,
              float4* __restrict__ Z, float* __restrict__ stats) {
  HF_PDL_ENTRY();
  constexpr int LPR = D / 4;
  constexpr int NS = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const int sl = lane % LPR, sid = lane / LPR;
  long long row = (long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int dh4 = (D / H) / 4;            // lanes per head
  const int h = sl / dh4;
  const int b = row_ptr[row], e = row_ptr[row + 1];
  const float sd = s_dst[row * H + h];
  float m = -INFINITY;
  for (int base = b; base < e; base += 32) {
    const int n = min(32, e - base);
    const int my_col = lane < n ? __ldg(col + base + lane) : 0;
    for (int k = 0; k < n; k += NS) {
      int idx = k + sid;
      int c = __shfl_sync(0xffffffffu, my_col, idx < n ? idx : 0);
      if (idx < n) m = fmaxf(m, att_logit<MUL>(__ldg(s_src + (long long)c * H + h), sd, slope));
    }
  }
  // all streams agree on the max
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int base = b; base < e; base += 32) {
    const int n = min(32, e - base);
    const int my_col = lane < n ? __ldg(col + base + lane) : 0;
    int k = 0;
    for (; k + NS * kUnroll <= n; k += NS * kUnroll) {
      float4 v[kUnroll];
      float sc[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        int c = __shfl_sync(0xffffffffu, my_col, k + u * NS + sid);
        v[u] = ldg4(Y + (long long)c * LPR + sl);
        sc[u] = __ldg(s_src + (long long)c * H + h);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        float p = expf(att_logit<MUL>(sc[u], sd, slope) - m);
        l += p;
        acc = f4fma(p, v[u], acc);
      }
    }
    for (; k < n; k += NS) {
      int idx = k + sid;
      int c = __shfl_sync(0xffffffffu, my_col, idx < n ? idx : 0);
      if (idx < n) {
        float p = expf(att_logit<MUL>(__ldg(s_src + (long long)c * H + h), sd, slope) - m);
        l += p;
        acc = f4fma(p, ldg4(Y + (long long)c * LPR + sl), acc);
      }
    }
  }
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) {
    acc = f4add(acc, f4shfl_xor(acc, o));
    l += __shfl_xor_sync(0xffffffffu, l, o);
  }
  if (sid == 0) {
    if (e > b) {
      acc = make_float4(__fdiv_rn(acc.x, l), __fdiv_rn(acc.y, l), __fdiv_rn(acc.z, l),
                        __fdiv_rn(acc.w, l));
    } else {
      m = 0.f;
      l = 0.f;
    }
    Z[row * LPR + sl] = acc;
    if (sl % dh4 == 0) {
      stats[row * 2 * H + h] = m;
      stats[row * 2 * H + H + h] = l;
    }
  }
}

// D = 64: one merged row per HALF warp (16 lanes x float4 = one Y row); the
// two halves process two rows independently (rows are short: ~3-10 edges).
// Same two passes as k_agg_fwd_gat; edges summed in row order.
template <bool MUL>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_fwd_gat_half(long long rows, int H, float slope, const int* __restrict__ row_ptr,
                   const int* __restrict__ col, const float4* __restrict__ Y,
                   const float* __restrict__ s_src, const float* __restrict__ s_dst,
                   float4* __restrict__ Z, float* __restrict__ stats) {
  HF_PDL_ENTRY();
  const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
  const unsigned mask = 0xffffu << (16 * half);
  const long long row = ((long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5)) * 2 + half;
  if (row >= rows) return;
  const int dh4 = (64 / H) / 4;
  const int h = hl / dh4;
  const int b = row_ptr[row], e = row_ptr[row + 1];
  const float sd = s_dst[row * H + h];
  float m = -INFINITY;
  for (int base = b; base < e; base += 16) {
    const int n = min(16, e - base);
    const int my_col = hl < n ? __ldg(col + base + hl) : 0;
    for (int k = 0; k < n; k++) {
      const int c = __shfl_sync(mask, my_col, k, 16);
      m = fmaxf(m, att_logit<MUL>(__ldg(s_src + (long long)c * H + h), sd, slope));
    }
  }
  float l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int base = b; base < e; base += 16) {
    const int n = min(16, e - base);
    const int my_col = hl < n ? __ldg(col + base + hl) : 0;
    int k = 0;
    for (; k + 4 <= n; k += 4) {
      float4 v[4];
      float sc[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int c = __shfl_sync(mask, my_col, k + u, 16);
        v[u] = ldg4(Y + (long long)c * 16 + hl);
        sc[u] = __ldg(s_src + (long long)c * H + h);
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const float p = expf(att_logit<MUL>(sc[u], sd, slope) - m);
        l += p;
        acc = f4fma(p, v[u], acc);
      }
    }
    for (; k < n; k++) {
      const int c = __shfl_sync(mask, my_col, k, 16);
      const float p = expf(att_logit<MUL>(__ldg(s_src + (long long)c * H + h), sd, slope) - m);
      l += p;
      acc = f4fma(p, ldg4(Y + (long long)c * 16 + hl), acc);
    }
  }
  if (e > b) {
    acc = make_float4(__fdiv_rn(acc.x, l), __fdiv_rn(acc.y, l), __fdiv_rn(acc.z, l),
                      __fdiv_rn(acc.w, l));
  } else {
    m = 0.f;
    l = 0.f;
  }
  Z[row * 16 + hl] = acc;
  if (hl % dh4 == 0) {
    stats[row * 2 * H + h] = m;
    stats[row * 2 * H + H + h] = l;
  }
}

// ---------------------------------------------------- backward SUM/MEAN (CSC)
// dY[u] = sum_{q in column u} w(row_q) G[row_q + shift(r(row_q))].
struct BwdMeta {
  int R;
  int shift[HF_MAX_R];   // type_dst_off[t(r)] - rel_row_off[r]
};

// Transpose SpMM of the sum / mean aggregation (the adjoint of Alg. 1):
//   dY[u] = sum_{p in CSC column u} w(m_p) G[g(m_p)],  m_p = csc_row[p],
// g(m) = m + shift[r(m)] the type-major G row of merged row m = (r, i), w = 1
// (sum) or 1 / |row m| (mean, reading C19: the product w*g is rounded, then
// summed, as an fp32 multiply followed by an add).  No pre-scaled copy of G:
// the lane that loads csc_row[p] resolves (g(m), w) -- relation by binary
// search over rel_row_off in shared memory, degree from row_ptr -- and
// broadcasts them to the lanes that gather the row.
__device__ __forceinline__ float4 f4mul_add(float w, float4 x, float4 a, bool mean) {
  if (!mean) return f4add(a, x);
  return make_float4(__fadd_rn(a.x, __fmul_rn(w, x.x)), __fadd_rn(a.y, __fmul_rn(w, x.y)),
                     __fadd_rn(a.z, __fmul_rn(w, x.z)), __fadd_rn(a.w, __fmul_rn(w, x.w)));
}

// Edge-balanced CSC walk.  Warp k owns the CSC entries [k E, (k+1) E) (E
// chosen per call), whatever columns they fall in, so a hub column costs no
// more per warp than a run of one-entry columns.  The build's csc_col gives
// every entry's column directly (no search over col_ptr): the warp walks its
// entries in sub-batches of 32 (coalesced loads of csc_col / csc_row, two
// sub-batches ahead; the mean's row_ptr pair one ahead), the lane of an entry
// resolves (g, w) and whether the entry closes its column's piece, and the
// whole warp gathers kEDepth G rows at a time (D/32 floats per lane), summing
// a column's rows in registers in CSC order.  A closed piece goes
//   - to dY when the column lies inside the chunk,
//   - to the chunk's head slot when the column began before the chunk
//     (head_col[k] records it), to its tail slot when it runs past the end
//     (tail_col[k]); the fix-up kernel adds tail[a] + head[a+1] + ... in chunk
//     order (deterministic).
// E is chosen per call (kEMin <= E <= kEMax) so that the chunks fill one
// wave of resident warps: small layers get short chunks (more warps, shorter
// dependent chains), large ones long chunks (fewer split columns).  Either
// way the chunk count is at most max(resident warps, N / kEMax) + 1, which
// sizes the partial slots of the workspace.
static constexpr int kEMin = 8, kEMax = 256;
static constexpr int kEDepth = 8;
static inline long long bwd_resident_warps() { return (long long)sm_count() * 3 * kWarpsPerBlock; }
static inline int bwd_chunk_entries(long long N) {
  const long long warps = bwd_resident_warps();          // resident at 3 blocks/SM
  return (int)std::max<long long>(kEMin, std::min<long long>(kEMax, (N + warps - 1) / warps));
}
static inline long long bwd_max_chunks(long long N) {
  return std::max(bwd_resident_warps(), (N + kEMax - 1) / kEMax) + 1;
}

template <int D> struct RowVec;
template <> struct RowVec<128> { using T = float4; };
template <> struct RowVec<64> { using T = float2; };
__device__ __forceinline__ float2 vzero(float2) { return make_float2(0.f, 0.f); }
__device__ __forceinline__ float4 vzero(float4) { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float2 vadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float4 vadd(float4 a, float4 b) { return f4add(a, b); }
__device__ __forceinline__ float2 vmul_add(float w, float2 x, float2 a, bool mean) {
  if (!mean) return vadd(a, x);
  return make_float2(__fadd_rn(a.x, __fmul_rn(w, x.x)), __fadd_rn(a.y, __fmul_rn(w, x.y)));
}
__device__ __forceinline__ float4 vmul_add(float w, float4 x, float4 a, bool mean) {
  return f4mul_add(w, x, a, mean);
}
__device__ __forceinline__ float2 vfma(float s, float2 y, float2 a) {
  return make_float2(fmaf(s, y.x, a.x), fmaf(s, y.y, a.y));
}
__device__ __forceinline__ float4 vfma(float s, float4 y, float4 a) { return f4fma(s, y, a); }
template <int D>
__device__ __forceinline__ typename RowVec<D>::T ldg_row(const float* p, int lane) {
  return __ldg(reinterpret_cast<const typename RowVec<D>::T*>(p) + lane);
}

// The chunk [p0, pend) and the columns of the entries just before and after it.
struct ChunkCtx {
  int p0, pend, prev_col, after_col;
};
// Column of the entry after mine (lane 31: first of the next sub-batch).
__device__ __forceinline__ int next_col(const ChunkCtx& cx, int q, int lane, int col_c,
                                        int col_n) {
  const int nx0 = __shfl_sync(0xffffffffu, col_n, 0);
  const int dn = __shfl_down_sync(0xffffffffu, col_c, 1);
  if (q + lane + 1 == cx.pend) return cx.after_col;
  return lane == 31 ? nx0 : dn;
}
// G row of merged row m: m + shift[r(m)], r by binary search of rel_row_off
__device__ __forceinline__ int g_row(int m, const int* s_roff, const int* s_shift, int R) {
  int lo = 0, hi = R;                                 // s_roff[lo] <= m < s_roff[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s_roff[mid] <= m) lo = mid; else hi = mid;
  }
  return m + s_shift[lo];
}

template <int D, bool MEAN>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 3)
k_agg_bwd_e(BwdMeta bm, const int* __restrict__ rel_row_off_d, const int* __restrict__ row_ptr,
            long long N, const int* __restrict__ csc_col, const int* __restrict__ csc_row,
            const typename RowVec<D>::T* __restrict__ G, typename RowVec<D>::T* __restrict__ dY,
            typename RowVec<D>::T* __restrict__ part, int* __restrict__ head_col,
            int* __restrict__ tail_col, int n_chunks, int E) {
  HF_PDL_ENTRY();
  using VT = typename RowVec<D>::T;
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ int s_roff[HF_MAX_R + 1];
  __shared__ int s_shift[HF_MAX_R];
  for (int i = threadIdx.x; i <= bm.R; i += blockDim.x) {
    s_roff[i] = rel_row_off_d[i];
    if (i < bm.R) s_shift[i] = bm.shift[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (k >= n_chunks) return;
  ChunkCtx cx;
  cx.p0 = k * E;
  cx.pend = (int)min(N, (long long)cx.p0 + E);
  cx.prev_col = cx.p0 > 0 ? __ldg(csc_col + cx.p0 - 1) : -1;
  cx.after_col = cx.pend < N ? __ldg(csc_col + cx.pend) : -1;
  const int p0 = cx.p0, pend = cx.pend;
  // software pipeline: csc_col / csc_row two sub-batches ahead, row_ptr one
  int col_c = p0 + lane < pend ? __ldg(csc_col + p0 + lane) : -1;
  int row_c = p0 + lane < pend ? __ldg(csc_row + p0 + lane) : -1;
  int rb_c = 0, re_c = 1;
  if (MEAN && row_c >= 0) { rb_c = __ldg(row_ptr + row_c); re_c = __ldg(row_ptr + row_c + 1); }
  int col_n = p0 + 32 + lane < pend ? __ldg(csc_col + p0 + 32 + lane) : -1;
  int row_n = p0 + 32 + lane < pend ? __ldg(csc_row + p0 + 32 + lane) : -1;
  const int c0 = __shfl_sync(FULL, col_c, 0);
  if (lane == 0) head_col[k] = c0 >= 0 && c0 == cx.prev_col ? c0 : -1;
  int tail = -1;
  VT acc = vzero(VT{});
#pragma unroll 1
  for (int q = p0; q < pend; q += 32) {
    const int n = __popc(__ballot_sync(FULL, col_c >= 0));      // valid entries: a prefix
    if (n == 0) break;
    const int nx = next_col(cx, q, lane, col_c, col_n);
    VT* my_dst = nullptr;
    if (col_c >= 0 && (nx != col_c || q + lane + 1 == pend)) {  // my entry closes a piece
      if (col_c == cx.prev_col) my_dst = part + 2ll * k * 32;             // head slot
      else if (nx == col_c) { my_dst = part + (2ll * k + 1) * 32; tail = col_c; }  // tail
      else my_dst = dY + (long long)col_c * 32;
    }
    const int qn = q + 32;
    const int col_nn = qn + 32 + lane < pend ? __ldg(csc_col + qn + 32 + lane) : -1;
    const int row_nn = qn + 32 + lane < pend ? __ldg(csc_row + qn + 32 + lane) : -1;
    int rb_n = 0, re_n = 1;
    if (MEAN && row_n >= 0) { rb_n = __ldg(row_ptr + row_n); re_n = __ldg(row_ptr + row_n + 1); }
    // (g, w) of my entry: G row m + shift[r(m)], weight 1 / |row m| (mean)
    const int my_g = row_c >= 0 ? g_row(row_c, s_roff, s_shift, bm.R) : 0;
    const float my_w = MEAN ? __frcp_rn((float)(re_c - rb_c)) : 1.f;
#pragma unroll 1
    for (int k0 = 0; k0 < n; k0 += kEDepth) {
      VT x[kEDepth];
#pragma unroll
      for (int j = 0; j < kEDepth; j++) {             // past n: entry n-1's row again
        const int g = __shfl_sync(FULL, my_g, min(k0 + j, n - 1));
        x[j] = __ldg(G + (long long)g * 32 + lane);
      }
#pragma unroll
      for (int j = 0; j < kEDepth; j++) {             // k0 + j <= 31
        VT* dst = reinterpret_cast<VT*>(
            __shfl_sync(FULL, reinterpret_cast<unsigned long long>(my_dst), k0 + j));
        if (MEAN) acc = vmul_add(__shfl_sync(FULL, my_w, k0 + j), x[j], acc, true);
        else acc = vadd(acc, x[j]);
        // past n the sum is garbage but never stored (dst null there): the
        // last valid entry closes its piece
        if (dst) {
          dst[lane] = acc;
          acc = vzero(VT{});
        }
      }
    }
    col_c = col_n; row_c = row_n; rb_c = rb_n; re_c = re_n;
    col_n = col_nn; row_n = row_nn;
  }
  tail = __reduce_max_sync(FULL, tail);
  if (lane == 0) tail_col[k] = tail;
}

// Number of chunks after k whose head slot continues column t (a hub column
// split over many short chunks): 32 head_col entries per ballot instead of one
// dependent load per chunk (the serial walk made the fix-up kernels the
// longest step of a small layer's backward: ~20 us on IMDB).
__device__ __forceinline__ int split_run(const int* __restrict__ head_col, int k, int n_chunks,
                                         int t, int lane) {
  int n = 0;
  for (int base = k + 1; base < n_chunks; base += 32) {
    const int j = base + lane;
    const unsigned b = __ballot_sync(0xffffffffu, j < n_chunks && __ldg(head_col + j) == t);
    if (b == 0xffffffffu) { n += 32; continue; }
    n += __ffs(~b) - 1;
    break;
  }
  return n;
}

// Split columns: dY[t] = tail[k] + head[k+1] + ... (chunk order).
template <int D>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_bwd_fix(const typename RowVec<D>::T* __restrict__ part, const int* __restrict__ head_col,
              const int* __restrict__ tail_col, typename RowVec<D>::T* __restrict__ dY,
              int n_chunks) {
  HF_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (k >= n_chunks) return;
  const int t = tail_col[k];
  if (t < 0) return;
  auto acc = part[(2ll * k + 1) * 32 + lane];
  const int n = split_run(head_col, k, n_chunks, t, lane);
#pragma unroll 4
  for (int j = k + 1; j <= k + n; j++) acc = vadd(acc, part[(2ll * j) * 32 + lane]);
  dY[(long long)t * 32 + lane] = acc;
}

// GAT pass 2 (CSC), edge-balanced like k_agg_bwd_e: per CSC entry p of column u
// (CSR position pos = csc_pos[p], merged row m = csc_row[p]) and head h,
//   dY[u]_h += alpha[pos, h] G[g(m)]_h     (fmaf, CSC order)
//   ds_src[u, h] += dpre[pos, h]
// and at the column's end dY[u] += ds_src[u] a_src(r(u)) (the scored form,
// att != NULL).  A lane holds D/32 features of one head; its alpha / dpre
// loads hit the same word as the other lanes of the head.  Split columns:
// (acc, dss) pieces in head / tail slots, k_agg_bwd_gat_fix adds them in
// chunk order and applies the a_src term.
static constexpr int kGatDss = 32;        // dss words per slot (H <= D/4 <= 32)
__device__ __forceinline__ int rel_of_y(int u, const int* s_yoff, int R) {
  int lo = 0, hi = R;                                 // s_yoff[lo] <= u < s_yoff[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s_yoff[mid] <= u) lo = mid; else hi = mid;
  }
  return lo;
}

template <int D>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 3)
k_agg_bwd_gat_e(BwdMeta bm, int H, const int* __restrict__ rel_row_off_d,
                const int* __restrict__ rel_y_off, long long N, const int* __restrict__ csc_col,
                const int* __restrict__ csc_pos, const int* __restrict__ csc_row,
                const float* __restrict__ alpha, const float* __restrict__ dpre,
                const float* __restrict__ Gf, float* __restrict__ dYf, float* __restrict__ ds_src,
                typename RowVec<D>::T* __restrict__ part, float* __restrict__ part_dss,
                int* __restrict__ head_col, int* __restrict__ tail_col, int n_chunks, int E,
                const float* __restrict__ att) {
  HF_PDL_ENTRY();
  using VT = typename RowVec<D>::T;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int VEC = D / 32;
  constexpr int kNone = -1, kHead = -2, kTail = -3;
  __shared__ int s_roff[HF_MAX_R + 1];
  __shared__ int s_yoff[HF_MAX_R + 1];
  __shared__ int s_shift[HF_MAX_R];
  for (int i = threadIdx.x; i <= bm.R; i += blockDim.x) {
    s_roff[i] = rel_row_off_d[i];
    s_yoff[i] = rel_y_off[i];
    if (i < bm.R) s_shift[i] = bm.shift[i];
  }
  __syncthreads();
  const VT* G = reinterpret_cast<const VT*>(Gf);
  VT* dY = reinterpret_cast<VT*>(dYf);
  const int lane = threadIdx.x & 31;
  const int dh = D / H;
  const int h = lane * VEC / dh;
  const bool head_lead = (lane * VEC) % dh == 0;
  const int k = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (k >= n_chunks) return;
  ChunkCtx cx;
  cx.p0 = k * E;
  cx.pend = (int)min(N, (long long)cx.p0 + E);
  cx.prev_col = cx.p0 > 0 ? __ldg(csc_col + cx.p0 - 1) : -1;
  cx.after_col = cx.pend < N ? __ldg(csc_col + cx.pend) : -1;
  const int p0 = cx.p0, pend = cx.pend;
  int col_c = p0 + lane < pend ? __ldg(csc_col + p0 + lane) : -1;
  int row_c = p0 + lane < pend ? __ldg(csc_row + p0 + lane) : -1;
  int pos_c = p0 + lane < pend ? __ldg(csc_pos + p0 + lane) : 0;
  int col_n = p0 + 32 + lane < pend ? __ldg(csc_col + p0 + 32 + lane) : -1;
  const int c0 = __shfl_sync(FULL, col_c, 0);
  if (lane == 0) head_col[k] = c0 >= 0 && c0 == cx.prev_col ? c0 : -1;
  int tail = -1;
  VT acc = vzero(VT{});
  float dss = 0.f;
#pragma unroll 1
  for (int q = p0; q < pend; q += 32) {
    const int n = __popc(__ballot_sync(FULL, col_c >= 0));
    if (n == 0) break;
    const int nx = next_col(cx, q, lane, col_c, col_n);
    int tgt = kNone;
    if (col_c >= 0 && (nx != col_c || q + lane + 1 == pend)) {
      if (col_c == cx.prev_col) tgt = kHead;
      else if (nx == col_c) { tgt = kTail; tail = col_c; }
      else tgt = col_c;
    }
    const int qn = q + 32;
    const int col_nn = qn + 32 + lane < pend ? __ldg(csc_col + qn + 32 + lane) : -1;
    const int row_n = qn + lane < pend ? __ldg(csc_row + qn + lane) : -1;
    const int pos_n = qn + lane < pend ? __ldg(csc_pos + qn + lane) : 0;
    const int my_g = row_c >= 0 ? g_row(row_c, s_roff, s_shift, bm.R) : 0;
#pragma unroll 1
    for (int k0 = 0; k0 < n; k0 += kEDepth) {
      VT x[kEDepth];
      float a[kEDepth], d[kEDepth];
#pragma unroll
      for (int j = 0; j < kEDepth; j++) {             // past n: entry n-1 again
        const int src = min(k0 + j, n - 1);
        const int g = __shfl_sync(FULL, my_g, src);
        const int ps = __shfl_sync(FULL, pos_c, src);
        x[j] = __ldg(G + (long long)g * 32 + lane);
        a[j] = __ldg(alpha + (long long)ps * H + h);
        d[j] = __ldg(dpre + (long long)ps * H + h);
      }
#pragma unroll
      for (int j = 0; j < kEDepth; j++) {             // k0 + j <= 31
        const int t = __shfl_sync(FULL, tgt, k0 + j);
        acc = vfma(a[j], x[j], acc);
        dss += d[j];
        if (t != kNone) {                             // warp-uniform
          if (t >= 0) {
            if (att)
              acc = vfma(dss, ldg_row<D>(att + (long long)rel_of_y(t, s_yoff, bm.R) * 2 * D, lane),
                         acc);
            dY[(long long)t * 32 + lane] = acc;
            if (head_lead) ds_src[(long long)t * H + h] = dss;
          } else {
            const long long sl = 2ll * k + (t == kTail);
            part[sl * 32 + lane] = acc;
            if (head_lead) part_dss[sl * kGatDss + h] = dss;
          }
          acc = vzero(VT{});
          dss = 0.f;
        }
      }
    }
    col_c = col_n; row_c = row_n; pos_c = pos_n;
    col_n = col_nn;
  }
  tail = __reduce_max_sync(FULL, tail);
  if (lane == 0) tail_col[k] = tail;
}

template <int D>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_bwd_gat_fix(int R, int H, const int* __restrict__ rel_y_off,
                  const typename RowVec<D>::T* __restrict__ part,
                  const float* __restrict__ part_dss, const int* __restrict__ head_col,
                  const int* __restrict__ tail_col, float* __restrict__ dYf,
                  float* __restrict__ ds_src, int n_chunks, const float* __restrict__ att) {
  HF_PDL_ENTRY();
  using VT = typename RowVec<D>::T;
  constexpr int VEC = D / 32;
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (k >= n_chunks) return;
  const int t = tail_col[k];
  if (t < 0) return;
  const int dh = D / H, h = lane * VEC / dh;
  VT acc = part[(2ll * k + 1) * 32 + lane];
  float dss = part_dss[(2ll * k + 1) * kGatDss + h];
  const int n = split_run(head_col, k, n_chunks, t, lane);
#pragma unroll 4
  for (int j = k + 1; j <= k + n; j++) {
    acc = vadd(acc, part[(2ll * j) * 32 + lane]);
    dss += part_dss[(2ll * j) * kGatDss + h];
  }
  if (att) {
    int lo = 0, hi = R;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(rel_y_off + mid) <= t) lo = mid; else hi = mid;
    }
    acc = vfma(dss, ldg_row<D>(att + (long long)lo * 2 * D, lane), acc);
  }
  reinterpret_cast<VT*>(dYf)[(long long)t * 32 + lane] = acc;
  if ((lane * VEC) % dh == 0) ds_src[(long long)t * H + h] = dss;
}

// ------------------------------------------------ backward GAT, pass 1 (rows)
// For row m=(r,i), head h, with g = G[g(m)] and alpha_p recomputed from stats:
//   dalpha_p = <g_h, Y[col_p]_h>,  za = sum_p alpha_p dalpha_p,
//   dpre_p   = alpha_p (dalpha_p - za) LeakyReLU'(pre_p),  ds_dst[m,h] = sum_p dpre_p.
// alpha and dpre are stored per CSR position for pass 2.
template <int D, bool MUL>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_bwd_gat_rows(BwdMeta bm, const int* __restrict__ rel_row_off_d, long long rows, int H,
                   float slope, const int* __restrict__ row_ptr, const int* __restrict__ col,
                   const float4* __restrict__ Y, const float* __restrict__ s_src,
                   const float* __restrict__ s_dst, const float* __restrict__ stats,
                   const float4* __restrict__ G, float* __restrict__ alpha,
                   float* __restrict__ dpre, float* __restrict__ ds_dst) {
  HF_PDL_ENTRY();
  constexpr int LPR = D / 4;
  constexpr int NS = 32 / LPR;
  __shared__ int s_roff[HF_MAX_R + 1];
  for (int i = threadIdx.x; i <= bm.R; i += blockDim.x) s_roff[i] = rel_row_off_d[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int sl = lane % LPR, sid = lane / LPR;
  long long row = (long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int dh4 = (D / H) / 4;
  const int h = sl / dh4;
  const bool head_lead = (sl % dh4) == 0;
  const int b = row_ptr[row], e = row_ptr[row + 1];
  if (e == b) {
    if (sid == 0 && head_lead) ds_dst[row * H + h] = 0.f;
    return;
  }
  const int r = upper_bound_i(s_roff, bm.R + 1, (int)row) - 1;
  const float4 g = ldg4(G + (row + bm.shift[r]) * LPR + sl);
  const float sd = s_dst[row * H + h];
  const float mx = stats[row * 2 * H + h];
  const float inv_l = 1.f / stats[row * 2 * H + H + h];
  float za = 0.f;
  for (int base = b; base < e; base += 32) {
    const int n = min(32, e - base);
    const int my_col = lane < n ? __ldg(col + base + lane) : 0;
    int k0 = 0;
    for (; k0 + NS * kUnroll <= n; k0 += NS * kUnroll) {
      // kUnroll edges per stream: loads first, then the dependent math
      float4 yv[kUnroll];
      float sv[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        const int idx = k0 + u * NS + sid;
        const int c = __shfl_sync(0xffffffffu, my_col, idx < n ? idx : 0);
        yv[u] = idx < n ? ldg4(Y + (long long)c * LPR + sl) : make_float4(0.f, 0.f, 0.f, 0.f);
        sv[u] = idx < n ? __ldg(s_src + (long long)c * H + h) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        const int idx = k0 + u * NS + sid;
        const float4 y = yv[u];
        float part = g.x * y.x + g.y * y.y + g.z * y.z + g.w * y.w;
        const float a = idx < n ? expf(att_logit<MUL>(sv[u], sd, slope) - mx) * inv_l : 0.f;
        for (int o = 1; o < dh4; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (idx < n) {
          za += a * part;
          if (head_lead) {
            alpha[(long long)(base + idx) * H + h] = a;
            dpre[(long long)(base + idx) * H + h] = part;   // dalpha, overwritten below
          }
        }
      }
    }
    for (int k = k0; k < n; k += NS) {
      int idx = k + sid;
      int c = __shfl_sync(0xffffffffu, my_col, idx < n ? idx : 0);
      float part = 0.f, a = 0.f;
      if (idx < n) {
        float4 y = ldg4(Y + (long long)c * LPR + sl);
        part = g.x * y.x + g.y * y.y + g.z * y.z + g.w * y.w;
        a = expf(att_logit<MUL>(__ldg(s_src + (long long)c * H + h), sd, slope) - mx) * inv_l;
      }
      for (int o = 1; o < dh4; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (idx < n) {
        za += a * part;
        if (head_lead) {
          alpha[(long long)(base + idx) * H + h] = a;
          dpre[(long long)(base + idx) * H + h] = part;   // dalpha, overwritten below
        }
      }
    }
  }
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) za += __shfl_xor_sync(0xffffffffu, za, o);
  __syncwarp();
  float dsd = 0.f;
  if (head_lead) {
    for (int p = b + sid; p < e; p += NS) {
      int c = __ldg(col + p);
      const float ss = __ldg(s_src + (long long)c * H + h);
      float a = alpha[(long long)p * H + h];
      float da = dpre[(long long)p * H + h];
      const float dl = a * (da - za);
      // dpre keeps the source-side partial (pass 2 sums it into ds_src)
      dpre[(long long)p * H + h] = dl * dlogit_dss<MUL>(ss, sd, slope);
      dsd += dl * dlogit_dsd<MUL>(ss, sd, slope);
    }
  }
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) dsd += __shfl_xor_sync(0xffffffffu, dsd, o);
  if (sid == 0 && head_lead) ds_dst[row * H + h] = dsd;
}

// D = 64: pass 1 with one merged row per HALF warp (rows are short; the
// warp-per-row form split each row over two streams).  Same arithmetic as
// k_agg_bwd_gat_rows, edges in row order.
template <bool MUL>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_bwd_gat_rows_half(BwdMeta bm, const int* __restrict__ rel_row_off_d, long long rows, int H,
                        float slope, const int* __restrict__ row_ptr,
                        const int* __restrict__ col, const float4* __restrict__ Y,
                        const float* __restrict__ s_src, const float* __restrict__ s_dst,
                        const float* __restrict__ stats, const float4* __restrict__ G,
                        float* __restrict__ alpha, float* __restrict__ dpre,
                        float* __restrict__ ds_dst) {
  HF_PDL_ENTRY();
  __shared__ int s_roff[HF_MAX_R + 1];
  for (int i = threadIdx.x; i <= bm.R; i += blockDim.x) s_roff[i] = rel_row_off_d[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
  const unsigned mask = 0xffffu << (16 * half);
  const long long row = ((long long)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5)) * 2 + half;
  if (row >= rows) return;
  const int dh4 = (64 / H) / 4;
  const int h = hl / dh4;
  const bool head_lead = (hl % dh4) == 0;
  const int b = row_ptr[row], e = row_ptr[row + 1];
  if (e == b) {
    if (head_lead) ds_dst[row * H + h] = 0.f;
    return;
  }
  const int r = upper_bound_i(s_roff, bm.R + 1, (int)row) - 1;
  const float4 g = ldg4(G + (row + bm.shift[r]) * 16 + hl);
  const float sd = s_dst[row * H + h];
  const float mx = stats[row * 2 * H + h];
  const float inv_l = 1.f / stats[row * 2 * H + H + h];
  float za = 0.f;
  for (int base = b; base < e; base += 16) {
    const int n = min(16, e - base);
    const int my_col = hl < n ? __ldg(col + base + hl) : 0;
    for (int k0 = 0; k0 < n; k0 += 4) {
      float4 yv[4];
      float sv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int idx = k0 + u;
        const int c = __shfl_sync(mask, my_col, idx < n ? idx : 0, 16);
        yv[u] = idx < n ? ldg4(Y + (long long)c * 16 + hl) : make_float4(0.f, 0.f, 0.f, 0.f);
        sv[u] = idx < n ? __ldg(s_src + (long long)c * H + h) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int idx = k0 + u;
        float part = g.x * yv[u].x + g.y * yv[u].y + g.z * yv[u].z + g.w * yv[u].w;
        for (int o = 1; o < dh4; o <<= 1) part += __shfl_xor_sync(mask, part, o, 16);
        if (idx < n) {
          const float a = expf(att_logit<MUL>(sv[u], sd, slope) - mx) * inv_l;
          za += a * part;
          if (head_lead) {
            alpha[(long long)(base + idx) * H + h] = a;
            dpre[(long long)(base + idx) * H + h] = part;   // dalpha, overwritten below
          }
        }
      }
    }
  }
  __syncwarp(mask);
  float dsd = 0.f;
  if (head_lead) {
    for (int p = b; p < e; p++) {
      const int c = __ldg(col + p);
      const float ss = __ldg(s_src + (long long)c * H + h);
      const float a = alpha[(long long)p * H + h];
      const float da = dpre[(long long)p * H + h];
      const float dl = a * (da - za);
      dpre[(long long)p * H + h] = dl * dlogit_dss<MUL>(ss, sd, slope);
      dsd += dl * dlogit_dsd<MUL>(ss, sd, slope);
    }
    ds_dst[row * H + h] = dsd;
  }
}

// ------------------------------------ GAT with the softmax across relations
// (reading C5'): the softmax of
// destination (t, i) runs over the union of its rows (r, i), t(r) = t, i.e.
// over all its in-edges whatever their relation; each row still receives its
// own edges' terms, so the semantic fusion's sum over r is the attention-
// weighted sum over all neighbours.  One warp per DESTINATION walks the rows
// of the relations into its type (relation order): pass 1 the max, pass 2 the
// normaliser, pass 3 each row's sum p Y / l.  stats (m, l) are written to
// every row of the destination, so the per-row backward machinery (pass 2 over
// the CSC) recomputes the same alpha.
struct XrelMeta {
  int T;
  int type_dst_off[HF_MAX_T + 1];
  int trel_off[HF_MAX_T + 1];     // relations into type t: trel_row[trel_off[t] .. trel_off[t+1])
  int trel_row[HF_MAX_R];         // rel_row_off[r] of those relations, ascending r
};

__device__ __forceinline__ int xrel_type(const XrelMeta& xm, int d) {
  int t = 0;
  while (t + 1 < xm.T && xm.type_dst_off[t + 1] <= d) t++;
  return t;
}

template <int D>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_fwd_gat_xrel(XrelMeta xm, int dst_rows, int H, float slope, const int* __restrict__ row_ptr,
                   const int* __restrict__ col, const float4* __restrict__ Y,
                   const float* __restrict__ s_src, const float* __restrict__ s_dst,
                   float4* __restrict__ Z, float* __restrict__ stats) {
  HF_PDL_ENTRY();
  constexpr int LPR = D / 4;
  constexpr int NS = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const int sl = lane % LPR, sid = lane / LPR;
  const int d = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (d >= dst_rows) return;
  const int t = xrel_type(xm, d);
  const int i = d - xm.type_dst_off[t];
  const int q0 = xm.trel_off[t], q1 = xm.trel_off[t + 1];
  const int dh4 = (D / H) / 4;
  const int h = sl / dh4;
  // pass 1: max of the logits over the union
  float m = -INFINITY;
  int deg = 0;
  for (int q = q0; q < q1; q++) {
    const long long row = (long long)xm.trel_row[q] + i;
    const int b = row_ptr[row], e = row_ptr[row + 1];
    deg += e - b;
    const float sd = s_dst[row * H + h];
    for (int p = b + sid; p < e; p += NS)
      m = fmaxf(m, leaky(__ldg(s_src + (long long)__ldg(col + p) * H + h) + sd, slope));
  }
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  // pass 2: normaliser
  float l = 0.f;
  for (int q = q0; q < q1; q++) {
    const long long row = (long long)xm.trel_row[q] + i;
    const int b = row_ptr[row], e = row_ptr[row + 1];
    const float sd = s_dst[row * H + h];
    for (int p = b + sid; p < e; p += NS)
      l += expf(leaky(__ldg(s_src + (long long)__ldg(col + p) * H + h) + sd, slope) - m);
  }
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  if (deg == 0) { m = 0.f; l = 0.f; }
  // pass 3: every row's share
  for (int q = q0; q < q1; q++) {
    const long long row = (long long)xm.trel_row[q] + i;
    const int b = row_ptr[row], e = row_ptr[row + 1];
    const float sd = s_dst[row * H + h];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int base = b; base < e; base += 32) {
      const int n = min(32, e - base);
      const int my_col = lane < n ? __ldg(col + base + lane) : 0;
      int k = 0;
      for (; k + NS * kUnroll <= n; k += NS * kUnroll) {
        float4 v[kUnroll];
        float sc[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; u++) {
          int c = __shfl_sync(0xffffffffu, my_col, k + u * NS + sid);
          v[u] = ldg4(Y + (long long)c * LPR + sl);
          sc[u] = __ldg(s_src + (long long)c * H + h);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; u++)
          acc = f4fma(expf(leaky(sc[u] + sd, slope) - m), v[u], acc);
      }
      for (; k < n; k += NS) {
        int idx = k + sid;
        int c = __shfl_sync(0xffffffffu, my_col, idx < n ? idx : 0);
        if (idx < n)
          acc = f4fma(expf(leaky(__ldg(s_src + (long long)c * H + h) + sd, slope) - m),
                      ldg4(Y + (long long)c * LPR + sl), acc);
      }
    }
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) acc = f4add(acc, f4shfl_xor(acc, o));
    if (sid == 0) {
      if (e > b)
        acc = make_float4(__fdiv_rn(acc.x, l), __fdiv_rn(acc.y, l), __fdiv_rn(acc.z, l),
                          __fdiv_rn(acc.w, l));
      Z[row * LPR + sl] = acc;
      if (sl % dh4 == 0) {
        stats[row * 2 * H + h] = m;
        stats[row * 2 * H + H + h] = l;
      }
    }
  }
}

// Backward pass 1, across relations: as k_agg_bwd_gat_rows, but
// za = sum alpha dalpha runs over the destination's union of rows (the fused
// output is the sum over them); g = G[d] is shared by all of its rows.
template <int D>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_agg_bwd_gat_xrel_dst(XrelMeta xm, int dst_rows, int H, float slope,
                       const int* __restrict__ row_ptr, const int* __restrict__ col,
                       const float4* __restrict__ Y, const float* __restrict__ s_src,
                       const float* __restrict__ s_dst, const float* __restrict__ stats,
                       const float4* __restrict__ G, float* __restrict__ alpha,
                       float* __restrict__ dpre, float* __restrict__ ds_dst) {
  HF_PDL_ENTRY();
  constexpr int LPR = D / 4;
  constexpr int NS = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const int sl = lane % LPR, sid = lane / LPR;
  const int d = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (d >= dst_rows) return;
  const int t = xrel_type(xm, d);
  const int i = d - xm.type_dst_off[t];
  const int q0 = xm.trel_off[t], q1 = xm.trel_off[t + 1];
  const int dh4 = (D / H) / 4;
  const int h = sl / dh4;
  const bool head_lead = (sl % dh4) == 0;
  const float4 g = ldg4(G + (long long)d * LPR + sl);
  float za = 0.f;
  for (int q = q0; q < q1; q++) {
    const long long row = (long long)xm.trel_row[q] + i;
    const int b = row_ptr[row], e = row_ptr[row + 1];
    if (e == b) continue;
    const float sd = s_dst[row * H + h];
    const float mx = stats[row * 2 * H + h];
    const float inv_l = 1.f / stats[row * 2 * H + H + h];
    for (int base = b; base < e; base += 32) {
      const int n = min(32, e - base);
      const int my_col = lane < n ? __ldg(col + base + lane) : 0;
      for (int k = 0; k < n; k += NS) {
        int idx = k + sid;
        int c = __shfl_sync(0xffffffffu, my_col, idx < n ? idx : 0);
        float part = 0.f, a = 0.f;
        if (idx < n) {
          float4 y = ldg4(Y + (long long)c * LPR + sl);
          part = g.x * y.x + g.y * y.y + g.z * y.z + g.w * y.w;
          a = expf(leaky(__ldg(s_src + (long long)c * H + h) + sd, slope) - mx) * inv_l;
        }
        for (int o = 1; o < dh4; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (idx < n) {
          za += a * part;
          if (head_lead) {
            alpha[(long long)(base + idx) * H + h] = a;
            dpre[(long long)(base + idx) * H + h] = part;   // dalpha, overwritten below
          }
        }
      }
    }
  }
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) za += __shfl_xor_sync(0xffffffffu, za, o);
  __syncwarp();
  for (int q = q0; q < q1; q++) {
    const long long row = (long long)xm.trel_row[q] + i;
    const int b = row_ptr[row], e = row_ptr[row + 1];
    const float sd = s_dst[row * H + h];
    float dsd = 0.f;
    if (head_lead) {
      for (int p = b + sid; p < e; p += NS) {
        int c = __ldg(col + p);
        float pre = __ldg(s_src + (long long)c * H + h) + sd;
        float a = alpha[(long long)p * H + h];
        float da = dpre[(long long)p * H + h];
        float dp = a * (da - za) * (pre > 0.f ? 1.f : slope);
        dpre[(long long)p * H + h] = dp;
        dsd += dp;
      }
    }
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) dsd += __shfl_xor_sync(0xffffffffu, dsd, o);
    if (sid == 0 && head_lead) ds_dst[row * H + h] = dsd;
  }
}

static void make_xrel(const LayerMeta& m, XrelMeta* xm) {
  xm->T = m.T;
  int q = 0;
  for (int t = 0; t < m.T; t++) {
    xm->type_dst_off[t] = m.type_dst_off[t];
    xm->trel_off[t] = q;
    for (int r = 0; r < m.R; r++)
      if (m.rel_dst[r] == t) xm->trel_row[q++] = m.rel_row_off[r];
  }
  xm->type_dst_off[m.T] = m.type_dst_off[m.T];
  xm->trel_off[m.T] = q;
}

static bool heads_ok(int D, int H) {
  if (H <= 0 || D % H) return false;
  int dh = D / H;
  return dh % 4 == 0 && (dh & (dh - 1)) == 0;
}

}  // namespace hf

using namespace hf;

extern "C" {

hifuse_status hifuse_aggregate_fwd(const hifuse_csr* csr, int64_t rows, hifuse_agg agg, int D,
                                   int heads, float slope, const float* d_Y, const float* d_s_src,
                                   const float* d_s_dst, float* d_Z, float* d_stats,
                                   hifuse_stream_t stream) {
  if (!csr || rows < 0 || !csr->row_ptr || (rows > 0 && (!d_Z || !csr->col || !d_Y)))
    return HIFUSE_ERR_INVALID_ARG;
  if (D != 64 && D != 128) return HIFUSE_ERR_UNSUPPORTED;
  if (!aligned16(d_Y) || !aligned16(d_Z)) return HIFUSE_ERR_ALIGNMENT;
  cudaStream_t s = st(stream);
  unsigned grid = ceil_div(rows, kWarpsPerBlock);
  const int TB = kWarpsPerBlock * 32;
  if (agg == HIFUSE_AGG_GAT || agg == HIFUSE_AGG_GAT_XREL || agg == HIFUSE_AGG_GAT_MUL) {
    if (!heads_ok(D, heads)) return HIFUSE_ERR_UNSUPPORTED;
    if (rows > 0 && (!d_s_src || !d_s_dst || !d_stats)) return HIFUSE_ERR_INVALID_ARG;
#define HF_GATF(MM)                                                                             \
  if (D == 128)                                                                                 \
    HF_LAUNCH((k_agg_fwd_gat<128, MM>), grid, TB, 0, s, (long long)rows, heads, slope,          \
              csr->row_ptr, csr->col, (const float4*)d_Y, d_s_src, d_s_dst, (float4*)d_Z,       \
              d_stats);                                                                         \
  else                                                                                          \
    HF_LAUNCH(k_agg_fwd_gat_half<MM>, ceil_div(rows, kWarpsPerBlock * 2), TB, 0, s,             \
              (long long)rows, heads, slope, csr->row_ptr, csr->col, (const float4*)d_Y,        \
              d_s_src, d_s_dst, (float4*)d_Z, d_stats)
    if (agg == HIFUSE_AGG_GAT_MUL) { HF_GATF(true); } else { HF_GATF(false); }
#undef HF_GATF
  } else if (agg == HIFUSE_AGG_SUM || agg == HIFUSE_AGG_MEAN) {
    bool mean = agg == HIFUSE_AGG_MEAN;
#define HF_AGG(DD, MM)                                                                   \
  HF_LAUNCH((k_agg_fwd<DD, MM>), grid, TB, 0, s, (long long)rows, csr->row_ptr, csr->col, \
            (const float4*)d_Y, (float4*)d_Z)
    if (D == 128) { if (mean) HF_AGG(128, true); else HF_AGG(128, false); }
    else { if (mean) HF_AGG(64, true); else HF_AGG(64, false); }
#undef HF_AGG
  } else {
    return HIFUSE_ERR_INVALID_ARG;
  }
  return last_cuda();
}

size_t hifuse_aggregate_fuse_ws_bytes(const hifuse_layer_shape* shape) {
  LayerMeta m;
  if (make_meta(shape, &m) != HIFUSE_OK) return 0;
  return carve_bytes(m.dst_rows > 0 ? m.dst_rows : 1, 4);
}

hifuse_status hifuse_aggregate_fuse_fwd(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                        hifuse_agg agg, int D, hifuse_act act, const float* d_Y,
                                        const float* d_R0, const float* d_bias, float* d_Z,
                                        float* d_H, void* d_ws, size_t ws_bytes,
                                        hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (agg != HIFUSE_AGG_SUM && agg != HIFUSE_AGG_MEAN) return HIFUSE_ERR_UNSUPPORTED;
  if (D != 64 && D != 128) return HIFUSE_ERR_UNSUPPORTED;
  if (!csr || !csr->row_ptr || (m.rows > 0 && (!d_Z || !csr->col || !d_Y)) ||
      (m.dst_rows > 0 && !d_H))
    return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_Y) || !aligned16(d_Z) || !aligned16(d_R0) || !aligned16(d_bias) ||
      !aligned16(d_H))
    return HIFUSE_ERR_ALIGNMENT;
  if (ws_bytes < hifuse_aggregate_fuse_ws_bytes(shape) || !d_ws) return HIFUSE_ERR_WORKSPACE;
  FuseEpi f;
  memset(&f, 0, sizeof(f));
  f.R = m.R;
  f.relu = act == HIFUSE_ACT_RELU ? 1 : 0;
  for (int r = 0; r <= m.R; r++) f.rel_row_off[r] = m.rel_row_off[r];
  for (int r = 0; r < m.R; r++) f.rel_dst[r] = m.rel_dst[r];
  for (int t = 0; t <= m.T; t++) f.type_dst_off[t] = m.type_dst_off[t];
  int k = 0, no = 0;
  for (int t = 0; t < m.T; t++) {
    f.list_off[t] = k;
    for (int r = 0; r < m.R; r++)
      if (m.rel_dst[r] == t) f.rel_rows[k++] = m.rel_row_off[r];
    if (k == f.list_off[t] && m.n_dst[t] > 0) {      // no relation enters t
      f.orph_t[f.n_orph_types] = t;
      f.orph_off[f.n_orph_types++] = no;
      no += m.n_dst[t];
    }
  }
  f.list_off[m.T] = k;
  f.orph_off[f.n_orph_types] = no;
  f.n_orph = no;
  f.agg_blocks = ceil_div(m.rows, kWarpsPerBlock);
  const unsigned grid = f.agg_blocks + ceil_div(no, kWarpsPerBlock);
  cudaStream_t s = st(stream);
  const int TB = kWarpsPerBlock * 32;
  const bool mean = agg == HIFUSE_AGG_MEAN;
#define HF_AF(DD, MM)                                                                          \
  HF_LAUNCH((k_agg_fuse_fwd<DD, MM>), grid, TB, 0, s, (long long)m.rows, csr->row_ptr,         \
            csr->col, (const float4*)d_Y, (float4*)d_Z, f, (const float4*)d_R0,               \
            (const float4*)d_bias, (float4*)d_H, (int*)d_ws)
  if (D == 128) { if (mean) HF_AF(128, true); else HF_AF(128, false); }
  else { if (mean) HF_AF(64, true); else HF_AF(64, false); }
#undef HF_AF
  return last_cuda();
}

hifuse_status hifuse_aggregate_fwd_xrel(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                        int D, int heads, float slope, const float* d_Y,
                                        const float* d_s_src, const float* d_s_dst, float* d_Z,
                                        float* d_stats, hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (!csr || !csr->row_ptr) return HIFUSE_ERR_INVALID_ARG;
  if (D != 64 && D != 128) return HIFUSE_ERR_UNSUPPORTED;
  if (!heads_ok(D, heads)) return HIFUSE_ERR_UNSUPPORTED;
  if (m.rows > 0 && (!d_Z || !d_stats || !d_s_dst || (m.N > 0 && (!csr->col || !d_Y || !d_s_src))))
    return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_Y) || !aligned16(d_Z)) return HIFUSE_ERR_ALIGNMENT;
  XrelMeta xm;
  make_xrel(m, &xm);
  cudaStream_t s = st(stream);
  unsigned grid = ceil_div(m.dst_rows, kWarpsPerBlock);
  const int TB = kWarpsPerBlock * 32;
  if (D == 128)
    HF_LAUNCH(k_agg_fwd_gat_xrel<128>, grid, TB, 0, s, xm, m.dst_rows, heads, slope, csr->row_ptr,
              csr->col, (const float4*)d_Y, d_s_src, d_s_dst, (float4*)d_Z, d_stats);
  else
    HF_LAUNCH(k_agg_fwd_gat_xrel<64>, grid, TB, 0, s, xm, m.dst_rows, heads, slope, csr->row_ptr,
              csr->col, (const float4*)d_Y, d_s_src, d_s_dst, (float4*)d_Z, d_stats);
  return last_cuda();
}

size_t hifuse_aggregate_features_ws_bytes(const hifuse_layer_shape* shape) {
  LayerMeta m;
  if (make_meta(shape, &m) != HIFUSE_OK) return 0;
  return carve_bytes(m.N > 0 ? m.N : 1, 4);
}

hifuse_status hifuse_aggregate_features_fwd(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                            hifuse_agg agg, int K, const float* d_X,
                                            int64_t x_rows, const int32_t* d_gather_ids,
                                            float* d_Xagg, void* d_ws, size_t ws_bytes,
                                            hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (agg != HIFUSE_AGG_SUM && agg != HIFUSE_AGG_MEAN) return HIFUSE_ERR_UNSUPPORTED;
  if (K != 64 && K != 128) return HIFUSE_ERR_UNSUPPORTED;
  if (!csr || !csr->row_ptr || !csr->rel_y_off || x_rows < 0 || !d_Xagg ||
      (m.N > 0 && (!csr->col || !csr->y_src || !d_X)))
    return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_X) || !aligned16(d_Xagg)) return HIFUSE_ERR_ALIGNMENT;
  if (ws_bytes < hifuse_aggregate_features_ws_bytes(shape) || !d_ws) return HIFUSE_ERR_WORKSPACE;
  cudaStream_t s = st(stream);
  char* p = (char*)d_ws;
  int* col_x = carve<int>(p, m.N > 0 ? m.N : 1);
  RelOff ro;     // by value (no host->device copy: graph-capturable)
  for (int r = 0; r < m.R; r++) ro.v[r] = m.type_src_off[m.rel_src[r]];
  HF_LAUNCH(k_col_to_x, ceil_div(m.N, 256), 256, 0, s, m.N, m.R, csr->rel_y_off, ro, csr->col,
            csr->y_src, d_gather_ids, col_x);
  unsigned grid = ceil_div((long long)m.rows, kWarpsPerBlock);
  const int TB = kWarpsPerBlock * 32;
  const bool mean = agg == HIFUSE_AGG_MEAN;
#define HF_AGG(DD, MM)                                                                  \
  do { if (m.rows <= kLatRows)                                                          \
    HF_LAUNCH((k_agg_fwd<DD, MM, true, kLatUnroll>), grid, TB, 0, s, (long long)m.rows,  \
              csr->row_ptr, col_x, (const float4*)d_X, (float4*)d_Xagg);                \
  else                                                                                  \
    HF_LAUNCH((k_agg_fwd<DD, MM, true>), grid, TB, 0, s, (long long)m.rows, csr->row_ptr, col_x, \
              (const float4*)d_X, (float4*)d_Xagg); } while (0)
  if (K == 128) { if (mean) HF_AGG(128, true); else HF_AGG(128, false); }
  else { if (mean) HF_AGG(64, true); else HF_AGG(64, false); }
#undef HF_AGG
  return last_cuda();
}

hifuse_status hifuse_feature_cols(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                  const int32_t* d_gather_ids, int32_t* d_col_x,
                                  hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (!csr || !d_col_x || (m.N > 0 && !csr->col)) return HIFUSE_ERR_INVALID_ARG;
  if (!csr->y_src) {
    // X-row build (no Y numbering): col already is the source's row in X
    HF_LAUNCH(k_xrow_to_feat, ceil_div(m.N, 256), 256, 0, st(stream), m.N, csr->col,
              d_gather_ids, d_col_x);
    return last_cuda();
  }
  if (!csr->rel_y_off) return HIFUSE_ERR_INVALID_ARG;
  RelOff ro;
  for (int r = 0; r < m.R; r++) ro.v[r] = m.type_src_off[m.rel_src[r]];
  HF_LAUNCH(k_col_to_x, ceil_div(m.N, 256), 256, 0, st(stream), m.N, m.R, csr->rel_y_off, ro,
            csr->col, csr->y_src, d_gather_ids, d_col_x);
  return last_cuda();
}

hifuse_status hifuse_aggregate_features_cols(const hifuse_layer_shape* shape,
                                             const hifuse_csr* csr, hifuse_agg agg, int K,
                                             const float* d_X, int64_t x_rows,
                                             const int32_t* d_col_x, float* d_Xagg,
                                             hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (agg != HIFUSE_AGG_SUM && agg != HIFUSE_AGG_MEAN) return HIFUSE_ERR_UNSUPPORTED;
  if (K != 64 && K != 128) return HIFUSE_ERR_UNSUPPORTED;
  if (!csr || !csr->row_ptr || x_rows < 0 || !d_Xagg || (m.N > 0 && (!d_col_x || !d_X)))
    return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_X) || !aligned16(d_Xagg)) return HIFUSE_ERR_ALIGNMENT;
  cudaStream_t s = st(stream);
  unsigned grid = ceil_div((long long)m.rows, kWarpsPerBlock);
  const int TB = kWarpsPerBlock * 32;
  const bool mean = agg == HIFUSE_AGG_MEAN;
#define HF_AGG(DD, MM)                                                                  \
  do { if (m.rows <= kLatRows)                                                          \
    HF_LAUNCH((k_agg_fwd<DD, MM, true, kLatUnroll>), grid, TB, 0, s, (long long)m.rows,  \
              csr->row_ptr, d_col_x, (const float4*)d_X, (float4*)d_Xagg);              \
  else                                                                                  \
    HF_LAUNCH((k_agg_fwd<DD, MM, true>), grid, TB, 0, s, (long long)m.rows, csr->row_ptr, d_col_x, \
              (const float4*)d_X, (float4*)d_Xagg); } while (0)
  if (K == 128) { if (mean) HF_AGG(128, true); else HF_AGG(128, false); }
  else { if (mean) HF_AGG(64, true); else HF_AGG(64, false); }
#undef HF_AGG
  return last_cuda();
}

hifuse_status hifuse_aggregate_features_cols_bf16(const hifuse_layer_shape* shape,
                                                  const hifuse_csr* csr, hifuse_agg agg, int K,
                                                  const void* d_Xb, int64_t x_rows,
                                                  const int32_t* d_col_x,
                                                  const int32_t* d_gather_ids, float* d_Xagg,
                                                  float* d_Xdst, hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (agg != HIFUSE_AGG_SUM && agg != HIFUSE_AGG_MEAN) return HIFUSE_ERR_UNSUPPORTED;
  if (K != 64 && K != 128) return HIFUSE_ERR_UNSUPPORTED;
  if (!csr || !csr->row_ptr || x_rows < 0 || !d_Xagg ||
      (m.N > 0 && (!d_col_x || !d_Xb)) || (d_Xdst && m.dst_rows > 0 && !d_Xb))
    return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_Xb) || !aligned16(d_Xagg) || !aligned16(d_Xdst)) return HIFUSE_ERR_ALIGNMENT;
  cudaStream_t s = st(stream);
  const unsigned agg_blocks = ceil_div((long long)m.rows, kWarpsPerBlock);
  const int TB = kWarpsPerBlock * 32;
  DstConv dc;
  dc.T = m.T;
  int acc = 0;
  for (int t = 0; t < m.T; t++) {
    dc.n_dst[t] = m.n_dst[t];
    dc.dst_off[t] = acc;
    acc += m.n_dst[t];
  }
  dc.dst_off[m.T] = acc;
  for (int t = 0; t <= m.T; t++) dc.type_src_off[t] = m.type_src_off[t];
  const unsigned conv_blocks = d_Xdst ? ceil_div((long long)acc * (K / 8), TB) : 0;
  const bool mean = agg == HIFUSE_AGG_MEAN;
#define HF_AGGB(DD, MM, CS)                                                                   \
  HF_LAUNCH((k_agg_fwd_bf16<DD, MM, CS>), agg_blocks + conv_blocks, TB, 0, s, (long long)m.rows, \
            agg_blocks, csr->row_ptr, d_col_x, (const uint4*)d_Xb, (float4*)d_Xagg, dc,        \
            d_gather_ids, (float4*)d_Xdst)
  // gathered through the feature store's row ids: raw features (evict-first)
  const bool fs = d_gather_ids != nullptr;
  if (K == 128) {
    if (mean) { if (fs) HF_AGGB(128, true, true); else HF_AGGB(128, true, false); }
    else { if (fs) HF_AGGB(128, false, true); else HF_AGGB(128, false, false); }
  } else {
    if (mean) { if (fs) HF_AGGB(64, true, true); else HF_AGGB(64, true, false); }
    else { if (fs) HF_AGGB(64, false, true); else HF_AGGB(64, false, false); }
  }
#undef HF_AGGB
  return last_cuda();
}

size_t hifuse_aggregate_bwd_ws_bytes(const hifuse_layer_shape* shape, hifuse_agg agg, int heads) {
  LayerMeta m;
  if (make_meta(shape, &m) != HIFUSE_OK) return 0;
  // edge-balanced CSC pass: two partial slots (D <= 128 floats) per chunk,
  // the chunk's head and tail columns
  const long long nch = bwd_max_chunks(m.N);
  size_t b = carve_bytes(2 * nch * 128, 4) + 2 * carve_bytes(nch, 4);
  if (agg == HIFUSE_AGG_GAT || agg == HIFUSE_AGG_GAT_XREL || agg == HIFUSE_AGG_GAT_MUL)
    b += carve_bytes(2 * nch * kGatDss, 4) + 2 * carve_bytes((long long)m.N * heads, 4);
  return b;
}

static hifuse_status aggregate_bwd_impl(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                        hifuse_agg agg, int D, int heads, float slope,
                                        const float* d_G, const float* d_Y, const float* d_s_src,
                                        const float* d_s_dst, const float* d_stats,
                                        const float* d_att, float* d_dY, float* d_ds_src,
                                        float* d_ds_dst, void* d_ws, size_t ws_bytes,
                                        hifuse_stream_t stream, bool row_grad = false) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (!csr || !csr->col_ptr || !csr->csc_row || !csr->csc_col || !csr->U_dev || !csr->rel_y_off ||
      !d_dY || !d_G)
    return HIFUSE_ERR_INVALID_ARG;
  if (D != 64 && D != 128) return HIFUSE_ERR_UNSUPPORTED;
  if (!aligned16(d_G) || !aligned16(d_dY)) return HIFUSE_ERR_ALIGNMENT;
  if (ws_bytes < hifuse_aggregate_bwd_ws_bytes(shape, agg, heads) || !d_ws)
    return HIFUSE_ERR_WORKSPACE;
  // every host-side check before the first enqueue (an invalid call launches nothing)
  const bool gat = agg == HIFUSE_AGG_GAT || agg == HIFUSE_AGG_GAT_XREL ||
                   agg == HIFUSE_AGG_GAT_MUL;
  if (row_grad && agg == HIFUSE_AGG_GAT_XREL) return HIFUSE_ERR_UNSUPPORTED;
  if (gat) {
    if (!heads_ok(D, heads)) return HIFUSE_ERR_UNSUPPORTED;
    if (!d_Y || !d_s_src || !d_s_dst || !d_stats || !d_ds_src || !d_ds_dst || !csr->csc_pos ||
        !csr->row_ptr || !csr->col || !csr->rel_row_off)
      return HIFUSE_ERR_INVALID_ARG;
  } else if (agg == HIFUSE_AGG_SUM || agg == HIFUSE_AGG_MEAN) {
    if ((agg == HIFUSE_AGG_MEAN && !csr->row_ptr) || !csr->rel_row_off)
      return HIFUSE_ERR_INVALID_ARG;
  } else {
    return HIFUSE_ERR_INVALID_ARG;
  }
  cudaStream_t s = st(stream);
  BwdMeta bm;
  bm.R = m.R;
  // G row of merged row m: m + shift[r(m)] (type-major G), or m itself for a
  // per-merged-row gradient (row_grad: HAN fusion, hifuse_aggregate_bwd_rows)
  for (int r = 0; r < m.R; r++)
    bm.shift[r] = row_grad ? 0 : m.type_dst_off[m.rel_dst[r]] - m.rel_row_off[r];
  char* p = (char*)d_ws;
  const int TB = kWarpsPerBlock * 32;
  // edge-balanced CSC pass: chunks of E entries, two partial slots per chunk
  const int E = bwd_chunk_entries(m.N);
  const long long nch = (m.N + E - 1) / E, nch_max = bwd_max_chunks(m.N);
  const unsigned gridE = ceil_div(nch, kWarpsPerBlock);
  float* part = carve<float>(p, 2 * nch_max * 128);
  int* head_col = carve<int>(p, nch_max);
  int* tail_col = carve<int>(p, nch_max);
  if (gat) {
    float* part_dss = carve<float>(p, 2 * nch_max * kGatDss);
    float* alpha = carve<float>(p, (long long)m.N * heads);
    float* dpre = carve<float>(p, (long long)m.N * heads);
    unsigned gridR = ceil_div(m.rows, kWarpsPerBlock);
    XrelMeta xm;
    if (agg == HIFUSE_AGG_GAT_XREL) make_xrel(m, &xm);
#define HF_GAT(DD, MM)                                                                         \
  if (agg == HIFUSE_AGG_GAT_XREL)                                                              \
    HF_LAUNCH(k_agg_bwd_gat_xrel_dst<DD>, ceil_div(m.dst_rows, kWarpsPerBlock), TB, 0, s, xm, \
              m.dst_rows, heads, slope, csr->row_ptr, csr->col, (const float4*)d_Y, d_s_src,   \
              d_s_dst, d_stats, (const float4*)d_G, alpha, dpre, d_ds_dst);                    \
  else if (DD == 64)                                                                           \
    HF_LAUNCH(k_agg_bwd_gat_rows_half<MM>, ceil_div(m.rows, kWarpsPerBlock * 2), TB, 0, s, bm,  \
              csr->rel_row_off, (long long)m.rows, heads, slope, csr->row_ptr, csr->col,        \
              (const float4*)d_Y, d_s_src, d_s_dst, d_stats, (const float4*)d_G, alpha, dpre,   \
              d_ds_dst);                                                                       \
  else                                                                                         \
    HF_LAUNCH((k_agg_bwd_gat_rows<DD, MM>), gridR, TB, 0, s, bm, csr->rel_row_off,              \
              (long long)m.rows,                                                              \
              heads, slope, csr->row_ptr, csr->col, (const float4*)d_Y, d_s_src, d_s_dst,     \
              d_stats, (const float4*)d_G, alpha, dpre, d_ds_dst);                            \
  HF_LAUNCH(k_agg_bwd_gat_e<DD>, gridE, TB, 0, s, bm, heads, csr->rel_row_off, csr->rel_y_off,    \
            (long long)m.N, csr->csc_col, csr->csc_pos, csr->csc_row, alpha, dpre, d_G, d_dY,   \
            d_ds_src, (RowVec<DD>::T*)part, part_dss, head_col, tail_col, (int)nch, E, d_att);  \
  HF_LAUNCH(k_agg_bwd_gat_fix<DD>, gridE, TB, 0, s, m.R, heads, csr->rel_y_off,                   \
            (const RowVec<DD>::T*)part, part_dss, head_col, tail_col, d_dY, d_ds_src, (int)nch, \
            d_att)
    const bool mul = agg == HIFUSE_AGG_GAT_MUL;
    if (D == 128) { if (mul) { HF_GAT(128, true); } else { HF_GAT(128, false); } }
    else { if (mul) { HF_GAT(64, true); } else { HF_GAT(64, false); } }
#undef HF_GAT
  } else {
#define HF_BWD(DD, MM)                                                                        \
  HF_LAUNCH((k_agg_bwd_e<DD, MM>), gridE, TB, 0, s, bm, csr->rel_row_off, csr->row_ptr,          \
            (long long)m.N, csr->csc_col, csr->csc_row, (const RowVec<DD>::T*)d_G,              \
            (RowVec<DD>::T*)d_dY, (RowVec<DD>::T*)part, head_col, tail_col, (int)nch, E);       \
  HF_LAUNCH((k_agg_bwd_fix<DD>), gridE, TB, 0, s, (const RowVec<DD>::T*)part, head_col,          \
            tail_col, (RowVec<DD>::T*)d_dY, (int)nch)
    bool mean = agg == HIFUSE_AGG_MEAN;
    if (D == 128) { if (mean) { HF_BWD(128, true); } else { HF_BWD(128, false); } }
    else { if (mean) { HF_BWD(64, true); } else { HF_BWD(64, false); } }
#undef HF_BWD
  }
  return last_cuda();
}

hifuse_status hifuse_aggregate_bwd(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                   hifuse_agg agg, int D, int heads, float slope,
                                   const float* d_G, const float* d_Y, const float* d_s_src,
                                   const float* d_s_dst, const float* d_stats, float* d_dY,
                                   float* d_ds_src, float* d_ds_dst, void* d_ws, size_t ws_bytes,
                                   hifuse_stream_t stream) {
  return aggregate_bwd_impl(shape, csr, agg, D, heads, slope, d_G, d_Y, d_s_src, d_s_dst, d_stats,
                            nullptr, d_dY, d_ds_src, d_ds_dst, d_ws, ws_bytes, stream);
}

hifuse_status hifuse_aggregate_bwd_scored(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                          hifuse_agg agg, int D, int heads, float slope,
                                          const float* d_G, const float* d_Y,
                                          const float* d_s_src, const float* d_s_dst,
                                          const float* d_stats, const float* d_att, float* d_dY,
                                          float* d_ds_src, float* d_ds_dst, void* d_ws,
                                          size_t ws_bytes, hifuse_stream_t stream) {
  if ((agg != HIFUSE_AGG_GAT && agg != HIFUSE_AGG_GAT_XREL && agg != HIFUSE_AGG_GAT_MUL) ||
      !d_att)
    return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_att)) return HIFUSE_ERR_ALIGNMENT;
  return aggregate_bwd_impl(shape, csr, agg, D, heads, slope, d_G, d_Y, d_s_src, d_s_dst, d_stats,
                            d_att, d_dY, d_ds_src, d_ds_dst, d_ws, ws_bytes, stream);
}

hifuse_status hifuse_aggregate_bwd_rows(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                        hifuse_agg agg, int D, int heads, float slope,
                                        const float* d_dZ, const float* d_Y,
                                        const float* d_s_src, const float* d_s_dst,
                                        const float* d_stats, const float* d_att, float* d_dY,
                                        float* d_ds_src, float* d_ds_dst, void* d_ws,
                                        size_t ws_bytes, hifuse_stream_t stream) {
  if (d_att && (agg == HIFUSE_AGG_SUM || agg == HIFUSE_AGG_MEAN)) return HIFUSE_ERR_INVALID_ARG;
  if (d_att && !aligned16(d_att)) return HIFUSE_ERR_ALIGNMENT;
  return aggregate_bwd_impl(shape, csr, agg, D, heads, slope, d_dZ, d_Y, d_s_src, d_s_dst,
                            d_stats, d_att, d_dY, d_ds_src, d_ds_dst, d_ws, ws_bytes, stream,
                            true);
}

}  // extern "C"

// project.cu -- A2+A3 feature projection and its backward.
//
// Groups: relation r (rows = the relation's compact Y rows, A = X_{s(r)} rows
// gathered through y_src; B = W_rel[r]) and root type t (rows = the
// destination prefix of type t, A = X_t rows, B = W_root[t]).  Layer 0 reads
// A rows straight from the type-major global feature store through
// gather_ids, so feature collection (A2, the paper's "reorganize and retrieve
// features" kernel, line 219) is fused into the projection's A loads.
//
// This file holds the CUDA-core fp32 path (HIFUSE_PREC_FP32) and the
// backward; the tcgen05 TF32 forward lives in project_tc.cu.
#include <cstdlib>
#include "project.cuh"

namespace hf {

// ------------------------------------------------------------ group table --
// tile_off[g] = first tile of group g (tiles of kBM rows), chunk_off[g] =
// first wgrad chunk (kCH rows); groups: R relations then T root types.
__global__ void k_group_table(ProjMeta pm, const int* __restrict__ rel_y_off, int* tile_off,
                              int* chunk_off, int BM, int CH) {
  HF_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  int t_acc = 0, c_acc = 0;
  for (int g = 0; g < pm.R + pm.T; g++) {
    int rows = g < pm.R ? rel_y_off[g + 1] - rel_y_off[g] : (pm.has_root ? pm.n_dst[g - pm.R] : 0);
    tile_off[g] = t_acc;
    chunk_off[g] = c_acc;
    t_acc += (rows + BM - 1) / BM;
    c_acc += (rows + CH - 1) / CH;
  }
  tile_off[pm.R + pm.T] = t_acc;
  chunk_off[pm.R + pm.T] = c_acc;
}

// Resolves tile/chunk `bid` to (group, first local row, row count).
__device__ __forceinline__ bool resolve(const ProjMeta& pm, const int* table, const int* rel_y_off,
                                        int bid, int step, int* g_out, int* r0, int* nrows) {
  int G = pm.R + pm.T;
  if (bid >= table[G]) return false;
  int lo = 0, hi = G;   // last g with table[g] <= bid
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (table[mid] <= bid) lo = mid; else hi = mid;
  }
  // skip empty groups sharing the same start
  while (lo + 1 < G && table[lo + 1] <= bid) lo++;
  int g = lo;
  int total = g < pm.R ? rel_y_off[g + 1] - rel_y_off[g] : pm.n_dst[g - pm.R];
  int local0 = (bid - table[g]) * step;
  *g_out = g;
  *r0 = local0;
  *nrows = min(step, total - local0);
  return *nrows > 0;
}

// X row of the A operand for local row `j` of group g.
__device__ __forceinline__ long long a_row(const ProjMeta& pm, const int* rel_y_off,
                                           const int* y_src, const int* gather_ids, int g, int j) {
  int x;
  if (g < pm.R) x = pm.type_src_off[pm.rel_src[g]] + y_src[rel_y_off[g] + j];
  else x = pm.type_src_off[g - pm.R] + j;
  return gather_ids ? (long long)gather_ids[x] : (long long)x;
}

// ------------------------------------------------------ SIMT forward GEMM --
// Tile: kBM x D outputs, 256 threads, each 4 rows x (D/16) cols, BK = 32.
template <int K, int D>
__global__ void __launch_bounds__(256)
k_proj_fwd_simt(ProjMeta pm, const int* __restrict__ tile_off, const int* __restrict__ rel_y_off,
                const int* __restrict__ y_src, const int* __restrict__ gather_ids,
                const float* __restrict__ X, const float* __restrict__ W_rel,
                const float* __restrict__ W_root, float* __restrict__ Y, float* __restrict__ R0) {
  HF_PDL_ENTRY();
  constexpr int BM = kBM, BK = 32, TN = D / 16;
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][D];
  int g, r0, nrows;
  if (!resolve(pm, tile_off, rel_y_off, blockIdx.x, BM, &g, &r0, &nrows)) return;
  const int tid = threadIdx.x;
  const float* W = g < pm.R ? W_rel + (long long)g * K * D : W_root + (long long)(g - pm.R) * K * D;
  // A rows this thread loads: tid/8 and tid/8 + 32
  long long xr[2];
#pragma unroll
  for (int i = 0; i < 2; i++) {
    int rr = tid / 8 + 32 * i;
    xr[i] = rr < nrows ? a_row(pm, rel_y_off, y_src, gather_ids, g, r0 + rr) : -1;
  }
  const int ty = tid / 16, tx = tid % 16;
  float acc[4][TN];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < TN; j++) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 2; i++) {
      int rr = tid / 8 + 32 * i, k4 = tid % 8;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (xr[i] >= 0) v = __ldg(reinterpret_cast<const float4*>(X + xr[i] * K + k0) + k4);
      As[k4 * 4 + 0][rr] = v.x;
      As[k4 * 4 + 1][rr] = v.y;
      As[k4 * 4 + 2][rr] = v.z;
      As[k4 * 4 + 3][rr] = v.w;
    }
#pragma unroll
    for (int i = 0; i < BK * D / 4 / 256; i++) {
      int idx = tid + 256 * i;
      int kr = idx / (D / 4), c4 = idx % (D / 4);
      *reinterpret_cast<float4*>(&Bs[kr][c4 * 4]) =
          __ldg(reinterpret_cast<const float4*>(W + (long long)(k0 + kr) * D) + c4);
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; kk++) {
      float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      float av[4] = {a.x, a.y, a.z, a.w};
      float bv[TN];
#pragma unroll
      for (int j = 0; j < TN / 4; j++) {
        float4 b = *reinterpret_cast<const float4*>(&Bs[kk][j * 64 + tx * 4]);
        bv[j * 4 + 0] = b.x; bv[j * 4 + 1] = b.y; bv[j * 4 + 2] = b.z; bv[j * 4 + 3] = b.w;
      }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* out = g < pm.R ? Y + (long long)rel_y_off[g] * D
                        : R0 + (long long)pm.type_dst_off[g - pm.R] * D;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int rr = ty * 4 + i;
    if (rr >= nrows) continue;
#pragma unroll
    for (int j = 0; j < TN / 4; j++)
      *reinterpret_cast<float4*>(out + (long long)(r0 + rr) * D + j * 64 + tx * 4) =
          make_float4(acc[i][j * 4], acc[i][j * 4 + 1], acc[i][j * 4 + 2], acc[i][j * 4 + 3]);
  }
}

// ---------------------------------------------------------- RGAT scores ----
// v[r][k][h] = sum_c W_r[k, h dh + c] a_dst[r, h, c]   (reading C7 fold)
__global__ void k_att_fold(int R, int K, int D, int H, const float* __restrict__ W_rel,
                           const float* __restrict__ att, float* __restrict__ v) {
  HF_PDL_ENTRY();
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * K * H) return;
  int h = idx % H, k = (idx / H) % K, r = idx / (H * K);
  int dh = D / H;
  const float* w = W_rel + ((long long)r * K + k) * D + h * dh;
  const float* a = att + (long long)r * 2 * D + D + h * dh;
  float s = 0.f;
  for (int c = 0; c < dh; c++) s = fmaf(w[c], a[c], s);
  v[idx] = s;
}

// s_src[u,h] = <Y[u, head h], a_src[r(u), head h]>, one warp per Y row.
__global__ void k_scores_src(int R, int D, int H, const int* __restrict__ U_dev,
                             const int* __restrict__ rel_y_off, const float* __restrict__ Y,
                             const float* __restrict__ att, float* __restrict__ s_src) {
  HF_PDL_ENTRY();
  __shared__ int s_yoff[HF_MAX_R + 1];
  for (int i = threadIdx.x; i <= R; i += blockDim.x) s_yoff[i] = rel_y_off[i];
  __syncthreads();
  int u = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (u >= *U_dev) return;
  int r = upper_bound_i(s_yoff, R + 1, u) - 1;
  const float* a = att + (long long)r * 2 * D;
  int dh = D / H;
  for (int h = 0; h < H; h++) {
    float s = 0.f;
    for (int c = lane; c < dh; c += 32) s = fmaf(Y[(long long)u * D + h * dh + c], a[h * dh + c], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) s_src[(long long)u * H + h] = s;
  }
}

// s_dst[(r,i),h] = <X_{t(r)}[i], v[r][:,h]>: one warp per merged row; the
// 32 lanes are (head h, K-chunk c) pairs, 32/H lanes per head, so each load
// instruction touches only 32/H X segments and 32/H contiguous v rows
// (v[r] is [K][H]); the chunk partials of a head meet by xor shuffles.
// (Thread-per-(row, head) with a serial 128-long K loop was latency-bound
// and, on its side branch, longer than the projection itself.)
template <int K, int HMAX>
__global__ void __launch_bounds__(256)
k_scores_dst(ProjMeta pm, int H, const int* __restrict__ gather_ids,
             const float* __restrict__ X, const float* __restrict__ v,
             float* __restrict__ s_dst) {
  HF_PDL_ENTRY();
  (void)HMAX;
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= pm.rows) return;
  const int lph = 32 / H;                    // lanes per head (H divides 32)
  const int h = lane / lph, c = lane % lph;
  const int kc = K / lph;                    // features per lane
  const int r = upper_bound_i(pm.rel_row_off, pm.R + 1, row) - 1;
  const int t = pm.rel_dst[r];
  const int x = pm.type_src_off[t] + (row - pm.rel_row_off[r]);
  const long long xr = gather_ids ? (long long)gather_ids[x] : (long long)x;
  const float* xp = X + xr * K + c * kc;
  const float* vp = v + ((long long)r * K + c * kc) * H + h;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  int k = 0;
  for (; k + 4 <= kc; k += 4) {
    a0 = fmaf(__ldg(xp + k), __ldg(vp + (k) * H), a0);
    a1 = fmaf(__ldg(xp + k + 1), __ldg(vp + (k + 1) * H), a1);
    a2 = fmaf(__ldg(xp + k + 2), __ldg(vp + (k + 2) * H), a2);
    a3 = fmaf(__ldg(xp + k + 3), __ldg(vp + (k + 3) * H), a3);
  }
  for (; k < kc; k++) a0 = fmaf(__ldg(xp + k), __ldg(vp + k * H), a0);
  float p = (a0 + a1) + (a2 + a3);
  for (int o = lph >> 1; o; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
  if (c == 0) s_dst[(long long)row * H + h] = p;
}

// H <= 8: warp per 2 consecutive merged rows (K = 64: both in one step,
// half a warp each).  The relation's folded weights v[r] ([K][H], <= 4 KB) are
// staged once per relation change into shared memory TRANSPOSED ([H][K]), so
// lane l reads the weights of its features 4l..4l+3 as one conflict-free
// 16-byte load per head; its X features are one coalesced 16-byte load; H
// partial dots are summed over the row's lanes by a butterfly.  (Reading
// v[r][4l..4l+3][0..H) from global per lane made every load instruction
// touch 32 lines: 30 us on IMDB vs 12 for the lane-per-(head, K-chunk) loop.)
constexpr int kSdRowsPerWarp = 2;   // (8: latency-bound chains of 8 dependent row loads)

template <int K, int H>
__global__ void __launch_bounds__(256)
k_scores_dst_v(ProjMeta pm, const int* __restrict__ gather_ids, const float* __restrict__ X,
               const float* __restrict__ v, float* __restrict__ s_dst) {
  HF_PDL_ENTRY();
  constexpr int LPR = K / 4, RPW = 32 / LPR;
  __shared__ __align__(16) float vT[8][H * K];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, sl = lane % LPR;
  float* my = vT[w];
  const int row0 = (blockIdx.x * 8 + w) * kSdRowsPerWarp;
  int r_cur = -1;
  for (int it = 0; it < kSdRowsPerWarp; it += RPW) {
    const int row = row0 + it + lane / LPR;
    const int rr = row < pm.rows ? row : pm.rows - 1;
    if (row0 + it >= pm.rows) break;                           // warp-uniform
    const int r = upper_bound_i(pm.rel_row_off, pm.R + 1, rr) - 1;
    // (K = 64: the two half-warp rows may differ in relation only at a
    // boundary -- stage per half then; rare, handled by the generic path)
    const int r0w = __shfl_sync(0xffffffffu, r, 0);
    const bool uni = __all_sync(0xffffffffu, r == r0w);
    if (uni && r0w != r_cur) {
      __syncwarp();
      const float4* src = reinterpret_cast<const float4*>(v + (long long)r0w * K * H);
      for (int q = lane; q < K * H / 4; q += 32) {
        const float4 x = __ldg(src + q);
        const float e[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int c = 0; c < 4; c++) {
          const int idx = 4 * q + c;
          my[(idx % H) * K + idx / H] = e[c];
        }
      }
      __syncwarp();
      r_cur = r0w;
    }
    float acc[H];
    const int t = pm.rel_dst[r];
    const int x = pm.type_src_off[t] + (rr - pm.rel_row_off[r]);
    const long long xr = gather_ids ? (long long)gather_ids[x] : (long long)x;
    const float4 xv = __ldg(reinterpret_cast<const float4*>(X + xr * K) + sl);
#pragma unroll
    for (int h = 0; h < H; h++) {
      float4 wv;
      if (uni) {
        wv = *reinterpret_cast<const float4*>(my + h * K + 4 * sl);
      } else {
        const float* vp = v + ((long long)r * K + 4 * sl) * H + h;
        wv = make_float4(__ldg(vp), __ldg(vp + H), __ldg(vp + 2 * H), __ldg(vp + 3 * H));
      }
      float a = __fmul_rn(xv.x, wv.x);
      a = fmaf(xv.y, wv.y, a);
      a = fmaf(xv.z, wv.z, a);
      acc[h] = fmaf(xv.w, wv.w, a);
    }
#pragma unroll
    for (int o = LPR / 2; o; o >>= 1)
#pragma unroll
      for (int h = 0; h < H; h++) acc[h] += __shfl_xor_sync(0xffffffffu, acc[h], o);
    if (row < pm.rows && sl == 0)
#pragma unroll
      for (int h = 0; h < H; h++) s_dst[(long long)row * H + h] = acc[h];
  }
}

static void launch_scores_dst(const ProjMeta& pm, int rows, int K, int H,
                              const int* gather_ids, const float* X, const float* v,
                              float* s_dst, cudaStream_t s) {
#define HF_SV(KK, HH)                                                                   \
  HF_LAUNCH((k_scores_dst_v<KK, HH>), ceil_div(rows, 8 * kSdRowsPerWarp), 256, 0, s, pm, \
            gather_ids, X, v, s_dst)
  if (K == 128 && H == 8) { HF_SV(128, 8); return; }
  if (K == 64 && H == 8) { HF_SV(64, 8); return; }
  if (K == 128 && H == 4) { HF_SV(128, 4); return; }
  if (K == 64 && H == 4) { HF_SV(64, 4); return; }
  if (K == 128 && H == 1) { HF_SV(128, 1); return; }
  if (K == 64 && H == 1) { HF_SV(64, 1); return; }
#undef HF_SV
  const unsigned grid = ceil_div(rows, 8);
#define HF_SD(KK, HH) \
  HF_LAUNCH((k_scores_dst<KK, HH>), grid, 256, 0, s, pm, H, gather_ids, X, v, s_dst)
  if (K == 128) HF_SD(128, 1);
  else HF_SD(64, 1);
#undef HF_SD
}

// ------------------------------------------------------------- backward ----
// dYt = dY + ds_src (x) a_src  (score chain), in place, one thread per float4.
__global__ void __launch_bounds__(256)
k_dy_score(int R, int D, int H, const int* __restrict__ U_dev, const int* __restrict__ rel_y_off,
           const float* __restrict__ att, const float* __restrict__ ds_src, float4* __restrict__ dY) {
  HF_PDL_ENTRY();
  __shared__ int s_yoff[HF_MAX_R + 1];
  for (int i = threadIdx.x; i <= R; i += blockDim.x) s_yoff[i] = rel_y_off[i];
  __syncthreads();
  const int D4 = D / 4;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int u = (int)(idx / D4), c4 = (int)(idx % D4);
  if (u >= *U_dev) return;
  const int r = upper_bound_i(s_yoff, R + 1, u) - 1;
  const int dh = D / H, h = (c4 * 4) / dh;
  const float g = ds_src[(long long)u * H + h];
  const float4 a = __ldg(reinterpret_cast<const float4*>(att + (long long)r * 2 * D) + c4);
  float4 y = dY[idx];
  y.x = fmaf(g, a.x, y.x); y.y = fmaf(g, a.y, y.y); y.z = fmaf(g, a.z, y.z); y.w = fmaf(g, a.w, y.w);
  dY[idx] = y;
}

// wgrad partials: chunk c of group g: P[c][k][d] = sum_{rows} A[row][k] B[row][d]
// A = X rows (gathered), B = dYt rows (relations) or G rows (root types).
template <int K, int D>
__global__ void __launch_bounds__(256)
k_wgrad_partial(ProjMeta pm, const int* __restrict__ chunk_off, const int* __restrict__ rel_y_off,
                const int* __restrict__ y_src, const int* __restrict__ gather_ids,
                const float* __restrict__ X, const float* __restrict__ dY,
                const float* __restrict__ G, float* __restrict__ partial) {
  HF_PDL_ENTRY();
  constexpr int RB = 32, TM = K / 16, TN = D / 16;
  __shared__ __align__(16) float As[RB][K];
  __shared__ __align__(16) float Bs[RB][D];
  __shared__ long long s_xr[RB];
  int g, r0, nrows;
  if (!resolve(pm, chunk_off, rel_y_off, blockIdx.x, kCH, &g, &r0, &nrows)) return;
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const float* Bbase = g < pm.R ? dY + (long long)rel_y_off[g] * D
                                : G + (long long)pm.type_dst_off[g - pm.R] * D;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; i++)
#pragma unroll
    for (int j = 0; j < TN; j++) acc[i][j] = 0.f;
  for (int rb = 0; rb < nrows; rb += RB) {
    if (tid < RB) {
      int rr = rb + tid;
      s_xr[tid] = rr < nrows ? a_row(pm, rel_y_off, y_src, gather_ids, g, r0 + rr) : -1;
    }
    __syncthreads();
    for (int idx = tid; idx < RB * K / 4; idx += 256) {
      int rr = idx / (K / 4), c4 = idx % (K / 4);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (s_xr[rr] >= 0) v = __ldg(reinterpret_cast<const float4*>(X + s_xr[rr] * K) + c4);
      *reinterpret_cast<float4*>(&As[rr][c4 * 4]) = v;
    }
    for (int idx = tid; idx < RB * D / 4; idx += 256) {
      int rr = idx / (D / 4), c4 = idx % (D / 4);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rb + rr < nrows)
        v = __ldg(reinterpret_cast<const float4*>(Bbase + (long long)(r0 + rb + rr) * D) + c4);
      *reinterpret_cast<float4*>(&Bs[rr][c4 * 4]) = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < RB; rr++) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM / 4; i++) {
        float4 a = *reinterpret_cast<const float4*>(&As[rr][i * 64 + ty * 4]);
        av[i * 4] = a.x; av[i * 4 + 1] = a.y; av[i * 4 + 2] = a.z; av[i * 4 + 3] = a.w;
      }
#pragma unroll
      for (int j = 0; j < TN / 4; j++) {
        float4 b = *reinterpret_cast<const float4*>(&Bs[rr][j * 64 + tx * 4]);
        bv[j * 4] = b.x; bv[j * 4 + 1] = b.y; bv[j * 4 + 2] = b.z; bv[j * 4 + 3] = b.w;
      }
#pragma unroll
      for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* P = partial + (long long)blockIdx.x * K * D;
#pragma unroll
  for (int i = 0; i < TM; i++) {
    int k = (i / 4) * 64 + ty * 4 + (i % 4);
#pragma unroll
    for (int j = 0; j < TN / 4; j++)
      *reinterpret_cast<float4*>(P + (long long)k * D + j * 64 + tx * 4) =
          make_float4(acc[i][j * 4], acc[i][j * 4 + 1], acc[i][j * 4 + 2], acc[i][j * 4 + 3]);
  }
}

// dW[g] = sum of group g's chunk partials, in chunk order (deterministic).
// dv != nullptr: adds dW_r[k, d] += dv[r, h(d), k] a_dst[r, d] (unused by the
// library's calls: RGAT adds that term in k_att_dw, after the reduce).
__global__ void k_wgrad_reduce(int R, int T, int KD, const int* __restrict__ chunk_off,
                               const float4* __restrict__ partial, float4* __restrict__ dW_rel,
                               float4* __restrict__ dW_root, ProjMeta pm,
                               const int* __restrict__ rel_y_off, int CH,
                               const float* __restrict__ dv, const float* __restrict__ att,
                               int D, int H) {
  HF_PDL_ENTRY();
  // chunk table: from chunk_off (SIMT path) or rebuilt here from rel_y_off
  __shared__ int s_co[HF_MAX_R + HF_MAX_T + 1];
  if (!chunk_off) {
    // group chunk counts loaded in parallel (one thread per group), then
    // scanned from shared memory by thread 0 (a serial loop over global
    // loads here left the block waiting at the barrier: ncu, mag layer 0)
    const int GG = pm.R + pm.T;
    if ((int)threadIdx.x < GG) {
      const int g = threadIdx.x;
      const int rows = g < pm.R ? rel_y_off[g + 1] - rel_y_off[g] : (pm.has_root ? pm.n_dst[g - pm.R] : 0);
      s_co[g + 1] = (rows + CH - 1) / CH;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_co[0] = 0;
      for (int g = 1; g <= GG; g++) s_co[g] += s_co[g - 1];
    }
    __syncthreads();
    chunk_off = s_co;
  }
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int KD4 = KD / 4;
  int G = dW_root ? R + T : R;
  if (idx >= (long long)G * KD4) return;
  int g = (int)(idx / KD4), e = (int)(idx % KD4);
  // four independent accumulators (fixed pairing: deterministic)
  float4 s[4];
#pragma unroll
  for (int q = 0; q < 4; q++) s[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  int c0 = chunk_off[g], c1 = chunk_off[g + 1];
  int c = c0;
  for (; c + 4 <= c1; c += 4) {
#pragma unroll
    for (int q = 0; q < 4; q++) {
      float4 v = partial[(long long)(c + q) * KD4 + e];
      s[q].x += v.x; s[q].y += v.y; s[q].z += v.z; s[q].w += v.w;
    }
  }
  for (; c < c1; c++) {
    float4 v = partial[(long long)c * KD4 + e];
    s[0].x += v.x; s[0].y += v.y; s[0].z += v.z; s[0].w += v.w;
  }
  float4 t = make_float4((s[0].x + s[1].x) + (s[2].x + s[3].x), (s[0].y + s[1].y) + (s[2].y + s[3].y),
                         (s[0].z + s[1].z) + (s[2].z + s[3].z), (s[0].w + s[1].w) + (s[2].w + s[3].w));
  if (g < R && dv) {
    const int K = KD / D, k = (4 * e) / D, d0 = (4 * e) % D, dh = D / H;
    const float* ad = att + (long long)g * 2 * D + D + d0;
    const float* dvk = dv + (long long)g * H * K + k;
    t.x = fmaf(dvk[(long long)((d0 + 0) / dh) * K], ad[0], t.x);
    t.y = fmaf(dvk[(long long)((d0 + 1) / dh) * K], ad[1], t.y);
    t.z = fmaf(dvk[(long long)((d0 + 2) / dh) * K], ad[2], t.z);
    t.w = fmaf(dvk[(long long)((d0 + 3) / dh) * K], ad[3], t.w);
  }
  if (g < R) dW_rel[(long long)g * KD4 + e] = t;
  else dW_root[(long long)(g - R) * KD4 + e] = t;
}

// dgrad: dX[type s tile] = sum_{r: s(r)=s} dYt[slot_y(r,j)] W_r^T
//                          + [j < n_dst(s)] G_s[j] W_root,s^T
template <int K, int D>
__global__ void __launch_bounds__(256)
k_dgrad(DgradMeta dm, const int* __restrict__ slot_y, const float* __restrict__ dY,
        const float* __restrict__ G, const float* __restrict__ W_rel,
        const float* __restrict__ W_root, float* __restrict__ dX) {
  HF_PDL_ENTRY();
  constexpr int BM = kBM, BK = 32, TN = K / 16;
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][K];
  const int s = upper_bound_i(dm.tile_off, dm.T + 1, blockIdx.x) - 1;
  const int j0 = (blockIdx.x - dm.tile_off[s]) * BM;
  const int nrows = min(BM, dm.n_src[s] - j0);
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  float acc[4][TN];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < TN; j++) acc[i][j] = 0.f;
  const int nterm = dm.out_off[s + 1] - dm.out_off[s] + (dm.has_root ? 1 : 0);
  for (int term = 0; term < nterm; term++) {
    const bool root = term == dm.out_off[s + 1] - dm.out_off[s];
    const int r = root ? -1 : dm.out_rel[dm.out_off[s] + term];
    const float* W = root ? W_root + (long long)s * K * D : W_rel + (long long)r * K * D;
    // A rows: tid/8 + 32 i, columns k4
    long long arow[2];
#pragma unroll
    for (int i = 0; i < 2; i++) {
      int rr = tid / 8 + 32 * i;
      long long a = -1;
      if (rr < nrows) {
        int j = j0 + rr;
        if (root) a = j < dm.n_dst[s] ? (long long)dm.type_dst_off[s] + j : -1;
        else a = slot_y[dm.slot_off[r] + j];
      }
      arow[i] = a;
    }
    const float* A = root ? G : dY;
    for (int d0 = 0; d0 < D; d0 += BK) {
#pragma unroll
      for (int i = 0; i < 2; i++) {
        int rr = tid / 8 + 32 * i, k4 = tid % 8;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (arow[i] >= 0) v = __ldg(reinterpret_cast<const float4*>(A + arow[i] * D + d0) + k4);
        As[k4 * 4 + 0][rr] = v.x;
        As[k4 * 4 + 1][rr] = v.y;
        As[k4 * 4 + 2][rr] = v.z;
        As[k4 * 4 + 3][rr] = v.w;
      }
      // Bs[dd][k] = W[k][d0 + dd]
      for (int idx = tid; idx < BK * K; idx += 256) {
        int k = idx / BK, dd = idx % BK;
        Bs[dd][k] = __ldg(W + (long long)k * D + d0 + dd);
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < BK; kk++) {
        float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        float av[4] = {a.x, a.y, a.z, a.w};
        float bv[TN];
#pragma unroll
        for (int j = 0; j < TN / 4; j++) {
          float4 b = *reinterpret_cast<const float4*>(&Bs[kk][j * 64 + tx * 4]);
          bv[j * 4] = b.x; bv[j * 4 + 1] = b.y; bv[j * 4 + 2] = b.z; bv[j * 4 + 3] = b.w;
        }
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int j = 0; j < TN; j++) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
  float* out = dX + (long long)dm.type_src_off[s] * K;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int rr = ty * 4 + i;
    if (rr >= nrows) continue;
#pragma unroll
    for (int j = 0; j < TN / 4; j++)
      *reinterpret_cast<float4*>(out + (long long)(j0 + rr) * K + j * 64 + tx * 4) =
          make_float4(acc[i][j * 4], acc[i][j * 4 + 1], acc[i][j * 4 + 2], acc[i][j * 4 + 3]);
  }
}

// RGAT attention-vector partials over chunks of kCH rows of one relation:
//   src (mode 0): P[c][h][w] = sum_u ds_src[u,h] Y[u,w]          rows = Y rows of r
//   dst (mode 1): P[c][h][w] = sum_i ds_dst[(r,i),h] X_t(r)[i][w] rows = merged rows of r
// Thread (h, w4) accumulates one float4 of the H x W outer-product sum; every
// row is read once per block (coalesced float4 rows), 4 rows in flight.
#ifndef HF_CHA
#define HF_CHA 32
#endif
static constexpr int kCHA = HF_CHA;    // attention-gradient chunk rows

// chunk table of kCHA-row chunks per relation into shared memory (warp 0)
__device__ __forceinline__ void att_chunk_table(int R, const int* ro, int* s_tab) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  int carry = 0;
  for (int base = 0; base < R; base += 32) {
    const int r = base + lane;
    const int t = r < R ? (ro[r + 1] - ro[r] + kCHA - 1) / kCHA : 0;
    int inc = t;
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += n;
    }
    if (r < R) s_tab[r] = carry + inc - t;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) s_tab[R] = carry;
}

__global__ void __launch_bounds__(1024)
k_att_partial(int R, int H, int W, int mode, const int* __restrict__ unused,
              const int* __restrict__ row_off, const float* __restrict__ A,
              const float* __restrict__ B, ProjMeta pm, const int* __restrict__ gather_ids,
              float* __restrict__ partial) {
  HF_PDL_ENTRY();
  __shared__ int s_tab[HF_MAX_R + 1];
  const int* ro = mode == 1 ? pm.rel_row_off : row_off;   // merged rows: host-known offsets
  att_chunk_table(R, ro, s_tab);
  __syncthreads();
  const int c = blockIdx.x;
  if (c >= s_tab[R]) return;
  const int r = upper_bound_i(s_tab, R + 1, c) - 1;
  const int first = ro[r] + (c - s_tab[r]) * kCHA;
  const int last = min(first + kCHA, ro[r + 1]);
  const int W4 = W / 4;
  const int h = threadIdx.x / W4, w4 = threadIdx.x % W4;
  if (h >= H) return;
  auto brow = [&](int row) -> long long {
    if (mode == 0) return row;
    const int x = pm.type_src_off[pm.rel_dst[r]] + (row - pm.rel_row_off[r]);
    return gather_ids ? (long long)gather_ids[x] : (long long)x;
  };
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int row = first;
  for (; row + 8 <= last; row += 8) {
    float a[8];
    float4 bv[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      a[q] = __ldg(A + (long long)(row + q) * H + h);
      bv[q] = __ldg(reinterpret_cast<const float4*>(B + brow(row + q) * W) + w4);
    }
#pragma unroll
    for (int q = 0; q < 8; q++) {
      acc.x = fmaf(a[q], bv[q].x, acc.x); acc.y = fmaf(a[q], bv[q].y, acc.y);
      acc.z = fmaf(a[q], bv[q].z, acc.z); acc.w = fmaf(a[q], bv[q].w, acc.w);
    }
  }
  for (; row < last; row++) {
    const float a = __ldg(A + (long long)row * H + h);
    const float4 bv = __ldg(reinterpret_cast<const float4*>(B + brow(row) * W) + w4);
    acc.x = fmaf(a, bv.x, acc.x); acc.y = fmaf(a, bv.y, acc.y);
    acc.z = fmaf(a, bv.z, acc.z); acc.w = fmaf(a, bv.w, acc.w);
  }
  reinterpret_cast<float4*>(partial + ((long long)c * H + h) * W)[w4] = acc;
}


// dv and datt of the RGAT attention chain in one kernel on the attention
// branch: block per (relation r, 32 consecutive d), 256 threads:
//   dv[r][h][k] for the block's heads: chunk sums of Pdst, the 8 warps
//               splitting the chunks, partials met in warp order (also
//               written to global for k_att_dw),
//   datt[r,0,d] = sum_chunks Psrc, datt[r,1,d] = sum_k W_r[k,d] dv[h(d)][k].
// (Formerly k_att_dv then k_att_da; merging all three final steps behind the
// weight-gradient reduce lengthened IMDB's input-layer call 31 -> 37 us: dv
// and datt only wait for the attention partials, k_att_dw for the reduce.)
__global__ void __launch_bounds__(256)
k_att_dvda(int R, int K, int D, int H, const int* __restrict__ rel_y_off, ProjMeta pm,
           const float* __restrict__ Psrc, const float* __restrict__ Pdst,
           const float* __restrict__ W_rel, float* __restrict__ datt, float* __restrict__ dv) {
  HF_PDL_ENTRY();
  __shared__ int s_tab[HF_MAX_R + 1], s_tab2[HF_MAX_R + 1];
  __shared__ float red[2][8][32];
  __shared__ float sdv[256];
  __shared__ float red2[8][256];
  const int tiles = D / 32;
  const int r = blockIdx.x / tiles, d0 = (blockIdx.x % tiles) * 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, d = d0 + lane;
  const int dh = D / H;
  const int h0 = d0 / dh, nh = (d0 + 31) / dh - h0 + 1;   // heads of the block's columns
  // chunk tables: source chunks (Y rows, rel_y_off) and destination chunks
  // (merged rows, host-known offsets); warp 0 builds both in turn
  att_chunk_table(R, pm.rel_row_off, s_tab2);
  __syncthreads();
  att_chunk_table(R, rel_y_off, s_tab);
  // dv of the block's heads: nh * K <= 256 contiguous values per chunk
  // (Pdst is [chunk][H][K]); the 8 warps split the relation's chunks, lane
  // owns values lane + 32 j, the warp partials meet in warp order
  {
    const int nv = nh * K;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; j++) acc[j] = 0.f;
    const float* pd = Pdst + (long long)h0 * K;
#pragma unroll 2
    for (int c = s_tab2[r] + w; c < s_tab2[r + 1]; c += 8) {
      const float* pc = pd + (long long)c * H * K;
#pragma unroll
      for (int j = 0; j < 8; j++)
        if (lane + 32 * j < nv) acc[j] += __ldg(pc + lane + 32 * j);
    }
#pragma unroll
    for (int j = 0; j < 8; j++) red2[w][lane + 32 * j] = acc[j];
  }
  __syncthreads();
  for (int o = threadIdx.x; o < nh * K; o += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int q = 0; q < 8; q++) t += red2[q][o];
    sdv[o] = t;
  }
  __syncthreads();
  const int h = d / dh;
  const float* vv = sdv + (h - h0) * K;
  // datt src half: the warp's chunks c0+w, +8, ... with four loads in flight
  // (fixed accumulator pairing: deterministic)
  float u;
  {
    const float* ps = Psrc + (long long)h * D + d;
    const long long cs = (long long)H * D;
    float u0 = 0.f, u1 = 0.f, u2 = 0.f, u3 = 0.f;
    int c = s_tab[r] + w;
    const int ce = s_tab[r + 1];
    for (; c + 24 < ce; c += 32) {
      u0 += ps[c * cs]; u1 += ps[(c + 8) * cs]; u2 += ps[(c + 16) * cs]; u3 += ps[(c + 24) * cs];
    }
    if (c < ce) u0 += ps[c * cs];
    if (c + 8 < ce) u1 += ps[(c + 8) * cs];
    if (c + 16 < ce) u2 += ps[(c + 16) * cs];
    u = (u0 + u1) + (u2 + u3);
  }
  float t = 0.f;
  const float* wp = W_rel + (long long)r * K * D + d;
  for (int k = w; k < K; k += 8) t = fmaf(wp[(long long)k * D], vv[k], t);
  red[0][w][lane] = u;
  red[1][w][lane] = t;
  // dv of the block's heads for k_att_dw (heads wider than 32 columns are
  // formed identically by each of their blocks: equal values written twice)
  for (int o = threadIdx.x; o < nh * K; o += blockDim.x)
    dv[((long long)r * H + h0) * K + o] = sdv[o];
  __syncthreads();
  if (w == 0) {
    float a = 0.f, b2 = 0.f;
#pragma unroll
    for (int q = 0; q < 8; q++) { a += red[0][q][lane]; b2 += red[1][q][lane]; }
    datt[(long long)r * 2 * D + d] = a;
    datt[(long long)r * 2 * D + D + d] = b2;
  }
}

// dW_r[k, d] += dv[r, h(d), k] a_dst[r, d]  (the s_dst chain's weight term,
// after the weight-gradient reduce wrote dW_rel)
__global__ void k_att_dw(int R, int K, int D, int H, const float* __restrict__ dv,
                         const float* __restrict__ att, float* __restrict__ dW_rel) {
  HF_PDL_ENTRY();
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)R * K * D) return;
  const int d = (int)(idx % D), k = (int)((idx / D) % K), r = (int)(idx / ((long long)K * D));
  const int h = d / (D / H);
  dW_rel[idx] += dv[((long long)r * H + h) * K + k] * att[(long long)r * 2 * D + D + d];
}

// dX_t[i] += sum_{r: t(r)=t} sum_h ds_dst[(r,i),h] v[r][:,h]   (s_dst chain);
// one thread per (destination row of the layer, k), relations in fixed order.
__global__ void k_dx_sdst(DgradMeta dm, int dst_rows, int K, int H, const float* __restrict__ v,
                          const float* __restrict__ ds_dst, float* __restrict__ dX) {
  HF_PDL_ENTRY();
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)dst_rows * K) return;
  int o = (int)(idx / K), k = (int)(idx % K);
  int t = upper_bound_i(dm.type_dst_off, dm.T + 1, o) - 1;
  int i = o - dm.type_dst_off[t];
  float s = 0.f;
  for (int q = dm.in_off[t]; q < dm.in_off[t + 1]; q++) {
    int r = dm.in_rel[q];
    long long row = dm.rel_row_off[r] + i;
    for (int h = 0; h < H; h++)
      s = fmaf(ds_dst[row * H + h], v[((long long)r * K + k) * H + h], s);
  }
  dX[(long long)(dm.type_src_off[t] + i) * K + k] += s;
}

void make_dgrad_meta(const LayerMeta& m, bool has_root, DgradMeta* dm, int bm) {
  dm->T = m.T;
  dm->has_root = has_root ? 1 : 0;
  dm->bm = bm;
  int tiles = 0, ko = 0, ki = 0;
  for (int t = 0; t < m.T; t++) {
    dm->tile_off[t] = tiles;
    tiles += (m.n_src[t] + bm - 1) / bm;
    dm->n_src[t] = m.n_src[t];
    dm->n_dst[t] = m.n_dst[t];
    dm->out_off[t] = ko;
    for (int r = 0; r < m.R; r++)
      if (m.rel_src[r] == t) dm->out_rel[ko++] = r;
    dm->in_off[t] = ki;
    for (int r = 0; r < m.R; r++)
      if (m.rel_dst[r] == t) dm->in_rel[ki++] = r;
  }
  dm->tile_off[m.T] = tiles;
  dm->out_off[m.T] = ko;
  dm->in_off[m.T] = ki;
  for (int t = 0; t <= m.T; t++) {
    dm->type_src_off[t] = m.type_src_off[t];
    dm->type_dst_off[t] = m.type_dst_off[t];
  }
  for (int r = 0; r <= m.R; r++) {
    dm->slot_off[r] = m.slot_off[r];
    dm->rel_row_off[r] = m.rel_row_off[r];
  }
}

void make_proj_meta(const LayerMeta& m, bool has_root, ProjMeta* pm) {
  pm->R = m.R;
  pm->T = m.T;
  pm->rows = m.rows;
  pm->has_root = has_root ? 1 : 0;
  for (int r = 0; r < m.R; r++) {
    pm->rel_src[r] = m.rel_src[r];
    pm->rel_dst[r] = m.rel_dst[r];
  }
  for (int r = 0; r <= m.R; r++) pm->rel_row_off[r] = m.rel_row_off[r];
  for (int t = 0; t < m.T; t++) pm->n_dst[t] = m.n_dst[t];
  for (int t = 0; t <= m.T; t++) {
    pm->type_src_off[t] = m.type_src_off[t];
    pm->type_dst_off[t] = m.type_dst_off[t];
  }
}

long long proj_max_tiles(const LayerMeta& m, int step) {
  long long U_max = m.N < m.S ? m.N : m.S;
  return (U_max + m.dst_rows) / step + m.R + m.T + 1;
}

}  // namespace hf

using namespace hf;

static bool kd_ok(int K, int D) { return (K == 64 || K == 128) && (D == 64 || D == 128); }

static bool heads_ok2(int D, int H) {
  if (H <= 0 || H > HIFUSE_MAX_HEADS || D % H) return false;
  int dh = D / H;
  return dh % 4 == 0 && (dh & (dh - 1)) == 0;
}

extern "C" {

size_t hifuse_project_ws_bytes(const hifuse_layer_shape* shape, int K, int D, int heads) {
  LayerMeta m;
  if (make_meta(shape, &m) != HIFUSE_OK) return 0;
  size_t b = 2 * carve_bytes(m.R + m.T + 1, 4);            // tile_off, chunk_off
  b += carve_bytes((long long)m.R * K * (heads > 0 ? heads : 1), 4);   // v
  b += carve_bytes((long long)(m.R + m.T) * K * D, 2);      // bf16 W^T (HIFUSE_PREC_BF16)
  return b;
}

static hifuse_status project_impl(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                  hifuse_layout layout, hifuse_prec prec, int K, int D, int heads,
                                  const float* d_X, int64_t x_rows, const int32_t* d_gather_ids,
                                  const float* d_W_rel, const float* d_W_root, const float* d_att,
                                  float* d_Y, uint16_t* d_Yb, float* d_R0, float* d_s_src,
                                  float* d_s_dst, void* d_ws, size_t ws_bytes,
                                  hifuse_stream_t stream) {
  if (layout != HIFUSE_LAYOUT_COMPACT) return HIFUSE_ERR_UNSUPPORTED;
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (!kd_ok(K, D)) return HIFUSE_ERR_UNSUPPORTED;
  if (!csr || !csr->rel_y_off || !csr->y_src || !csr->U_dev || !d_X || !d_W_rel ||
      (!d_Y && !d_Yb) || x_rows < 0 || (d_W_root && !d_R0))
    return HIFUSE_ERR_INVALID_ARG;
  if (d_att && (!heads_ok2(D, heads) || !d_s_src || !d_s_dst)) return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_X) || !aligned16(d_W_rel) || !aligned16(d_W_root) || !aligned16(d_Y) ||
      !aligned16(d_Yb) || !aligned16(d_R0))
    return HIFUSE_ERR_ALIGNMENT;
  // bf16 Y: the tcgen05 path without RGAT scores (RGCN)
  if (d_Yb && (d_att || (prec != HIFUSE_PREC_TF32 && prec != HIFUSE_PREC_BF16)))
    return HIFUSE_ERR_UNSUPPORTED;
  if (ws_bytes < hifuse_project_ws_bytes(shape, K, D, heads) || !d_ws) return HIFUSE_ERR_WORKSPACE;
  cudaStream_t s = st(stream);
  ProjMeta pm;
  make_proj_meta(m, d_W_root != nullptr, &pm);
  char* p = (char*)d_ws;
  int* tile_off = carve<int>(p, m.R + m.T + 1);
  int* chunk_off = carve<int>(p, m.R + m.T + 1);
  float* v = carve<float>(p, (long long)m.R * K * (heads > 0 ? heads : 1));
  uint16_t* wt = carve<uint16_t>(p, (long long)(m.R + m.T) * K * D);
  const bool tc = prec == HIFUSE_PREC_TF32 || prec == HIFUSE_PREC_BF16;
  // RGAT destination scores (v = W a_dst folded, s_dst = X v) only read X and
  // W: a parallel branch next to the projection GEMM (fp32 in every precision)
  Branch bs;
  bool sbr = false;
  if (d_att && tc) {
    sbr = branch_begin(s, &bs, 2);
    cudaStream_t sd = sbr ? bs.side : s;
    HF_LAUNCH(k_att_fold, ceil_div((long long)m.R * K * heads, 256), 256, 0, sd, m.R, K, D, heads,
              d_W_rel, d_att, v);
    launch_scores_dst(pm, m.rows, K, heads, d_gather_ids, d_X, v, d_s_dst, sd);
  }
  if (tc) {
    rc = project_tcp_launch(m, pm, K, D, csr->rel_y_off, csr->y_src, d_X, nullptr, d_gather_ids,
                            d_W_rel, d_W_root, d_Y, d_R0, d_att, d_s_src, heads, s,
                            prec == HIFUSE_PREC_BF16 ? wt : nullptr, d_Yb);   // s_src fused in the epilogue
    if (sbr) branch_end(s, bs);
    if (rc != HIFUSE_OK) return rc;
  } else if (prec == HIFUSE_PREC_FP32) {
    HF_LAUNCH(k_group_table, 1, 32, 0, s, pm, csr->rel_y_off, tile_off, chunk_off, kBM, kCH);
    unsigned grid = (unsigned)proj_max_tiles(m, kBM);
#define HF_FWD(KK, DD)                                                                    \
  HF_LAUNCH((k_proj_fwd_simt<KK, DD>), grid, 256, 0, s, pm, tile_off, csr->rel_y_off,     \
            csr->y_src, d_gather_ids, d_X, d_W_rel, d_W_root, d_Y, d_R0)
    if (K == 128 && D == 128) HF_FWD(128, 128);
    else if (K == 128 && D == 64) HF_FWD(128, 64);
    else if (K == 64 && D == 128) HF_FWD(64, 128);
    else HF_FWD(64, 64);
#undef HF_FWD
  } else {
    return HIFUSE_ERR_UNSUPPORTED;
  }
  if (d_att && !tc) {
    HF_LAUNCH(k_att_fold, ceil_div((long long)m.R * K * heads, 256), 256, 0, s, m.R, K, D, heads,
              d_W_rel, d_att, v);
    long long U_max = m.N < m.S ? m.N : m.S;
    HF_LAUNCH(k_scores_src, ceil_div(U_max, 8), 256, 0, s, m.R, D, heads, csr->U_dev,
              csr->rel_y_off, d_Y, d_att, d_s_src);
    launch_scores_dst(pm, m.rows, K, heads, d_gather_ids, d_X, v, d_s_dst, s);
  }
  return last_cuda();
}

hifuse_status hifuse_project(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                             hifuse_layout layout, hifuse_prec prec, int K, int D, int heads,
                             const float* d_X, int64_t x_rows, const int32_t* d_gather_ids,
                             const float* d_W_rel, const float* d_W_root, const float* d_att,
                             float* d_Y, float* d_R0, float* d_s_src, float* d_s_dst, void* d_ws,
                             size_t ws_bytes, hifuse_stream_t stream) {
  if (!d_Y) return HIFUSE_ERR_INVALID_ARG;
  return project_impl(shape, csr, layout, prec, K, D, heads, d_X, x_rows, d_gather_ids, d_W_rel,
                      d_W_root, d_att, d_Y, nullptr, d_R0, d_s_src, d_s_dst, d_ws, ws_bytes,
                      stream);
}

hifuse_status hifuse_project_y16(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                 hifuse_layout layout, hifuse_prec prec, int K, int D,
                                 const float* d_X, int64_t x_rows, const int32_t* d_gather_ids,
                                 const float* d_W_rel, const float* d_W_root, uint16_t* d_Yb,
                                 float* d_R0, void* d_ws, size_t ws_bytes,
                                 hifuse_stream_t stream) {
  if (!d_Yb) return HIFUSE_ERR_INVALID_ARG;
  return project_impl(shape, csr, layout, prec, K, D, 1, d_X, x_rows, d_gather_ids, d_W_rel,
                      d_W_root, nullptr, nullptr, d_Yb, d_R0, nullptr, nullptr, d_ws, ws_bytes,
                      stream);
}

size_t hifuse_project_bwd_ws_bytes(const hifuse_layer_shape* shape, int K, int D, int heads) {
  LayerMeta m;
  if (make_meta(shape, &m) != HIFUSE_OK) return 0;
  int H = heads > 0 ? heads : 1;
  long long chunks = proj_max_tiles(m, kCH < 128 ? kCH : 128);
  size_t b = 2 * carve_bytes(m.R + m.T + 1, 4);
  b += carve_bytes(chunks * K * D, 4);                       // wgrad partials
  b += carve_bytes((long long)m.R * K * H * 2, 4);           // v, dv
  b += 2 * carve_bytes(m.R + 1, 4);                          // att chunk tables
  long long U_max = m.N < m.S ? m.N : m.S;
  long long ach = U_max / 32 + m.rows / 32 + 2 * m.R + 2;
  b += carve_bytes(ach * H * (K > D ? K : D), 4) * 2;        // att partials
  b += carve_bytes(m.R + 1, 4);                              // host row table copy
  return b;
}

// The event ordering k_dx_sdst (dgrad branch) after the fold of W a_dst
// (source-side attention branch): owned by the caller's stream.
static cudaEvent_t fold_event(cudaStream_t s) {
  StreamCtx* c = stream_ctx(s);
  return c ? c->fold : nullptr;
}

static hifuse_status project_bwd_impl(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                      hifuse_layout layout, hifuse_prec prec, int K, int D,
                                      int heads, const float* d_X, int64_t x_rows,
                                      const int32_t* d_gather_ids, const float* d_W_rel,
                                      const float* d_W_root, const float* d_att,
                                      const float* d_Y, float* d_dY, const float* d_G,
                                      const float* d_ds_src, const float* d_ds_dst, float* d_dX,
                                      float* d_dW_rel, float* d_dW_root, float* d_datt,
                                      void* d_ws, size_t ws_bytes, hifuse_stream_t stream,
                                      bool scored) {
  if (layout != HIFUSE_LAYOUT_COMPACT) return HIFUSE_ERR_UNSUPPORTED;
  if (prec != HIFUSE_PREC_FP32 && prec != HIFUSE_PREC_TF32) return HIFUSE_ERR_UNSUPPORTED;
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (!kd_ok(K, D)) return HIFUSE_ERR_UNSUPPORTED;
  // d_dW_rel == NULL: input gradient only (RGCN; the caller runs the weight
  // gradient as a separate call, e.g. on a parallel stream)
  const bool wgrad = d_dW_rel != nullptr;
  // RGAT input gradient alone: only after hifuse_aggregate_bwd_scored (dY
  // already holds dYt, so the weights call does not apply the score chain twice)
  if (!csr || !d_X || !d_W_rel || !d_dY || x_rows < 0 || (!wgrad && (!d_dX || (d_att && !scored))) ||
      (d_W_root && (!d_G || (wgrad && !d_dW_root))))
    return HIFUSE_ERR_INVALID_ARG;
  if (d_att && (!heads_ok2(D, heads) || !d_ds_dst || (wgrad && (!d_ds_src || !d_datt || !d_Y))))
    return HIFUSE_ERR_INVALID_ARG;
  if (d_dX && d_gather_ids) return HIFUSE_ERR_UNSUPPORTED;
  if (ws_bytes < hifuse_project_bwd_ws_bytes(shape, K, D, heads) || !d_ws)
    return HIFUSE_ERR_WORKSPACE;
  cudaStream_t s = st(stream);
  ProjMeta pm;
  make_proj_meta(m, d_W_root != nullptr, &pm);
  int H = heads > 0 ? heads : 1;
  long long chunks = proj_max_tiles(m, kCH < 128 ? kCH : 128);
  char* p = (char*)d_ws;
  int* tile_off = carve<int>(p, m.R + m.T + 1);
  int* chunk_off = carve<int>(p, m.R + m.T + 1);
  float* partial = carve<float>(p, chunks * K * D);
  float* v = carve<float>(p, (long long)m.R * K * H * 2);
  int* src_chunk = carve<int>(p, m.R + 1);
  int* dst_chunk = carve<int>(p, m.R + 1);
  long long U_max = m.N < m.S ? m.N : m.S;
  long long ach = U_max / kCHA + m.rows / kCHA + 2 * m.R + 2;
  float* Psrc = carve<float>(p, ach * H * (K > D ? K : D));
  float* Pdst = carve<float>(p, ach * H * (K > D ? K : D));
  if (d_att && !scored) {      // scored: dY already holds dYt (hifuse_aggregate_bwd_scored)
    HF_LAUNCH(k_dy_score, ceil_div(U_max * (D / 4), 256), 256, 0, s, m.R, D, H, csr->U_dev,
              csr->rel_y_off, d_att, d_ds_src, (float4*)d_dY);
  }
  // dgrad (dX) is independent of the weight-gradient chain: it runs on a
  // parallel branch (the dYt it reads is final after k_dy_score)
  DgradMeta dm;
  if (!wgrad) {
    // RGAT: the s_dst chain's dX term needs v = W a_dst (weights only): the
    // fold runs on a parallel branch next to the dgrad, k_dx_sdst after both
    Branch bf;
    bool fbr = false;
    if (d_att) {
      fbr = branch_begin(s, &bf, 1);
      HF_LAUNCH(k_att_fold, ceil_div((long long)m.R * K * H, 256), 256, 0, fbr ? bf.side : s,
                m.R, K, D, H, d_W_rel, d_att, v);
    }
    if (prec == HIFUSE_PREC_TF32) {
      make_dgrad_meta(m, d_W_root != nullptr, &dm, 128);
      rc = dgrad_tc_launch(dm, K, D, csr->slot_y, d_dY, d_G, d_W_rel, d_W_root, d_dX, s, U_max,
                           m.R);
      if (fbr) branch_end(s, bf);
      if (rc != HIFUSE_OK) return rc;
      if (d_att)
        HF_LAUNCH(k_dx_sdst, ceil_div((long long)m.dst_rows * K, 256), 256, 0, s, dm,
                  m.dst_rows, K, H, v, d_ds_dst, d_dX);
      return last_cuda();
    }
    if (fbr) branch_end(s, bf);
    make_dgrad_meta(m, d_W_root != nullptr, &dm);
    unsigned gd = dm.tile_off[m.T];
#define HF_DG(KK, DD)                                                                         \
  HF_LAUNCH((k_dgrad<KK, DD>), gd, 256, 0, s, dm, csr->slot_y, d_dY, d_G, d_W_rel, d_W_root, d_dX)
    if (K == 128 && D == 128) HF_DG(128, 128);
    else if (K == 128 && D == 64) HF_DG(128, 64);
    else if (K == 64 && D == 128) HF_DG(64, 128);
    else HF_DG(64, 64);
#undef HF_DG
    if (d_att)
      HF_LAUNCH(k_dx_sdst, ceil_div((long long)m.dst_rows * K, 256), 256, 0, s, dm, m.dst_rows,
                K, H, v, d_ds_dst, d_dX);
    return last_cuda();
  }
  Branch br;
  bool branched = false;
  bool dx_sdst_done = false;
  if (d_dX && prec == HIFUSE_PREC_TF32) {
    make_dgrad_meta(m, d_W_root != nullptr, &dm, 128);
    branched = branch_begin(s, &br);
    rc = dgrad_tc_launch(dm, K, D, csr->slot_y, d_dY, d_G, d_W_rel, d_W_root, d_dX,
                         branched ? br.side : s, U_max, m.R);
    if (rc != HIFUSE_OK) {
      if (branched) branch_end(s, br);
      return rc;
    }
  }
  int CH = kCH;
  if (prec == HIFUSE_PREC_TF32) {
    CH = wgrad_chunk_rows(m);
    wgrad_tc_launch(m, pm, K, D, CH, chunk_off, csr->rel_y_off, csr->y_src, d_gather_ids, d_X,
                    d_dY, d_G, partial, (unsigned)proj_max_tiles(m, CH), s);
  } else {
    HF_LAUNCH(k_group_table, 1, 32, 0, s, pm, csr->rel_y_off, tile_off, chunk_off, kBM, kCH);
    unsigned grid = (unsigned)chunks;
#define HF_WG(KK, DD)                                                                          \
  HF_LAUNCH((k_wgrad_partial<KK, DD>), grid, 256, 0, s, pm, chunk_off, csr->rel_y_off,         \
            csr->y_src, d_gather_ids, d_X, d_dY, d_G, partial)
    if (K == 128 && D == 128) HF_WG(128, 128);
    else if (K == 128 && D == 64) HF_WG(128, 64);
    else if (K == 64 && D == 128) HF_WG(64, 128);
    else HF_WG(64, 64);
#undef HF_WG
  }
  int G = d_W_root ? m.R + m.T : m.R;
  // RGAT attention chain (independent of the wgrad partials until
  // k_att_dw adds into dW_rel): a second parallel branch
  Branch ba;
  bool abr = false;
  float* dvb = v + (long long)m.R * K * H;     // dv [R][H][K] after v in the workspace
  if (d_att) {
    // two parallel chains: (a) destination side: partials of ds_dst x X ->
    // dv; (b) source side: the fold v = W a_dst (for k_dx_sdst) and the
    // partials of ds_src x Y; (a) then waits for (b) and forms datt.
    abr = branch_begin(s, &ba, 1);
    cudaStream_t sa = abr ? ba.side : s;
    Branch bb;
    const bool bbr = abr && branch_begin(s, &bb, 3);
    cudaStream_t sb = bbr ? bb.side : sa;
    // v = W a_dst only feeds the dX term of the s_dst chain (no dX: input layer)
    if (d_dX)
      HF_LAUNCH(k_att_fold, ceil_div((long long)m.R * K * H, 256), 256, 0, sb, m.R, K, D, H,
                d_W_rel, d_att, v);
    // the s_dst chain's dX term needs only the fold and the dgrad: it runs on
    // the dgrad branch as soon as both are done (not after both attention
    // chains and k_att_dw)
    if (d_dX && branched && prec == HIFUSE_PREC_TF32) {
      cudaEvent_t ev = fold_event(s);
      if (ev) {
        cudaEventRecord(ev, sb);
        cudaStreamWaitEvent(br.side, ev, 0);
        HF_LAUNCH(k_dx_sdst, ceil_div((long long)m.dst_rows * K, 256), 256, 0, br.side, dm,
                  m.dst_rows, K, H, v, d_ds_dst, d_dX);
        dx_sdst_done = true;
      }
    }
    const unsigned gs = (unsigned)(U_max / kCHA + m.R + 1);
    const unsigned gdst = (unsigned)(m.rows / kCHA + m.R + 1);
    HF_LAUNCH(k_att_partial, gs, H * D / 4, 0, sb, m.R, H, D, 0, (const int*)nullptr,
              csr->rel_y_off, d_ds_src, d_Y, pm, d_gather_ids, Psrc);
    HF_LAUNCH(k_att_partial, gdst, H * K / 4, 0, sa, m.R, H, K, 1, (const int*)nullptr,
              (const int*)nullptr, d_ds_dst, d_X, pm, d_gather_ids, Pdst);
    if (bbr) {                          // (a) waits for (b)
      cudaEventRecord(bb.join, bb.side);
      cudaStreamWaitEvent(sa, bb.join, 0);
    }
    HF_LAUNCH(k_att_dvda, m.R * (D / 32), 256, 0, sa, m.R, K, D, H, csr->rel_y_off, pm, Psrc,
              Pdst, d_W_rel, d_datt, dvb);
  }
  // (the s_dst term dv (x) a_dst is added by k_att_dw after the join:
  // folding it into the reduce made the reduce wait for the attention branch,
  // measured +3 us per RGAT layer on IMDB)
  HF_LAUNCH(k_wgrad_reduce, ceil_div((long long)G * K * D / 4, 256), 256, 0, s, m.R, m.T, K * D,
            prec == HIFUSE_PREC_TF32 ? (const int*)nullptr : (const int*)chunk_off,
            (const float4*)partial, (float4*)d_dW_rel, (float4*)d_dW_root, pm, csr->rel_y_off, CH,
            (const float*)nullptr, (const float*)nullptr, 0, 1);
  if (d_att) {
    if (abr) branch_end(s, ba);
    HF_LAUNCH(k_att_dw, ceil_div((long long)m.R * K * D, 256), 256, 0, s, m.R, K, D, H, dvb, d_att,
              d_dW_rel);
  }
  if (branched) branch_end(s, br);       // join the dgrad branch
  if (d_dX) {
    if (prec == HIFUSE_PREC_TF32) {
      // launched above on the parallel branch
    } else {
      make_dgrad_meta(m, d_W_root != nullptr, &dm);
      unsigned gd = dm.tile_off[m.T];
#define HF_DG(KK, DD)                                                                         \
  HF_LAUNCH((k_dgrad<KK, DD>), gd, 256, 0, s, dm, csr->slot_y, d_dY, d_G, d_W_rel, d_W_root, d_dX)
      if (K == 128 && D == 128) HF_DG(128, 128);
      else if (K == 128 && D == 64) HF_DG(128, 64);
      else if (K == 64 && D == 128) HF_DG(64, 128);
      else HF_DG(64, 64);
#undef HF_DG
    }
    if (d_att && !dx_sdst_done)
      HF_LAUNCH(k_dx_sdst, ceil_div((long long)m.dst_rows * K, 256), 256, 0, s, dm, m.dst_rows, K,
                H, v, d_ds_dst, d_dX);
  }
  return last_cuda();
}

}  // extern "C"

// ------------------------------------------------ aggregate-first RGCN input --
// SURVEY §8(f) NEXT(3), "aggregate-then-project": for the linear RGCN message
// W_r x, Z_r = A_r (X W_r) = (A_r X) W_r exactly (linearity; PAPER.md's
// four-stage layer P:L112-125 with stages 2 and 3 swapped), so the input
// layer can aggregate raw features first (hifuse_aggregate_features_fwd) and
// project rho aggregated rows instead of U compact source rows.  The layer's
// backward needs no transpose SpMM: dW_r = Xagg_r^T G_t(r) (no dX for the
// input features).
static long long direct_max_chunks(const LayerMeta& m, int step) {
  return ((long long)m.rows + m.dst_rows) / step + m.R + m.T + 1;
}
// Row chunks of the aggregate-first layers' wgrad: one chunk per SM (each
// chunk writes a K x D partial that the reduce re-reads: 2 per SM doubled
// those bytes; measured on mag, project_aggregated_bwd.0 27.2 -> 24.5 us
// with 1, 35.3 us with 4)
#ifndef HF_DIRECT_CTAS_PER_SM
#define HF_DIRECT_CTAS_PER_SM 1
#endif
static int direct_chunk_rows(const LayerMeta& m) {
  long long ch = ((long long)m.rows + m.dst_rows) / (HF_DIRECT_CTAS_PER_SM * sm_count());
  ch = (ch + 31) / 32 * 32;
  return (int)(ch < 128 ? 128 : (ch > kCHT ? kCHT : ch));
}

extern "C" {

hifuse_status hifuse_project_aggregated(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                        hifuse_prec prec, int K, int D, const float* d_Xagg,
                                        const float* d_X, int64_t x_rows,
                                        const int32_t* d_gather_ids, const float* d_W_rel,
                                        const float* d_W_root, float* d_Z, float* d_R0,
                                        hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (!kd_ok(K, D) || prec != HIFUSE_PREC_TF32) return HIFUSE_ERR_UNSUPPORTED;
  if (!csr || !csr->rel_row_off || !d_Xagg || !d_W_rel || !d_Z || x_rows < 0 ||
      (d_W_root && (!d_R0 || !d_X)))
    return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_Xagg) || !aligned16(d_X) || !aligned16(d_W_rel) || !aligned16(d_W_root) ||
      !aligned16(d_Z) || !aligned16(d_R0))
    return HIFUSE_ERR_ALIGNMENT;
  ProjMeta pm;
  make_proj_meta(m, d_W_root != nullptr, &pm);
  rc = project_tcp_launch(m, pm, K, D, csr->rel_row_off, nullptr, d_X ? d_X : d_Xagg, d_Xagg,
                          d_gather_ids, d_W_rel, d_W_root, d_Z, d_R0, nullptr, nullptr, 1,
                          st(stream));
  if (rc != HIFUSE_OK) return rc;
  return last_cuda();
}

hifuse_status hifuse_project_fuse_aggregated(const hifuse_layer_shape* shape,
                                            const hifuse_csr* csr, hifuse_prec prec, int K, int D,
                                            hifuse_act act, const float* d_Xagg,
                                            const float* d_X, int64_t x_rows,
                                            const int32_t* d_gather_ids, const float* d_W_rel,
                                            const float* d_W_root, const float* d_bias,
                                            float* d_H, hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (!kd_ok(K, D) || prec != HIFUSE_PREC_TF32) return HIFUSE_ERR_UNSUPPORTED;
  if (act != HIFUSE_ACT_RELU && act != HIFUSE_ACT_NONE) return HIFUSE_ERR_INVALID_ARG;
  if (!csr || !csr->rel_row_off || !d_W_rel || (m.dst_rows > 0 && !d_H) || x_rows < 0 ||
      (m.rows > 0 && !d_Xagg) || (d_W_root && !d_X))
    return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_Xagg) || !aligned16(d_X) || !aligned16(d_W_rel) || !aligned16(d_W_root) ||
      !aligned16(d_bias) || !aligned16(d_H))
    return HIFUSE_ERR_ALIGNMENT;
  rc = fuse_gemm_launch(m, d_W_root != nullptr, K, D, act == HIFUSE_ACT_RELU, d_gather_ids, d_X,
                        d_Xagg, d_W_rel, d_W_root, d_bias, d_H, st(stream));
  if (rc != HIFUSE_OK) return rc;
  return last_cuda();
}

size_t hifuse_project_aggregated_bwd_ws_bytes(const hifuse_layer_shape* shape, int K, int D) {
  LayerMeta m;
  if (make_meta(shape, &m) != HIFUSE_OK) return 0;
  return carve_bytes(direct_max_chunks(m, 128) * K * D, 4);
}

hifuse_status hifuse_project_aggregated_bwd(const hifuse_layer_shape* shape,
                                            const hifuse_csr* csr, hifuse_prec prec, int K, int D,
                                            const float* d_Xagg, const float* d_X, int64_t x_rows,
                                            const int32_t* d_gather_ids, const float* d_G,
                                            float* d_dW_rel, float* d_dW_root, void* d_ws,
                                            size_t ws_bytes, hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (!kd_ok(K, D) || prec != HIFUSE_PREC_TF32) return HIFUSE_ERR_UNSUPPORTED;
  if (!csr || !csr->rel_row_off || !d_Xagg || !d_G || !d_dW_rel || x_rows < 0 ||
      (d_dW_root && !d_X))
    return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_Xagg) || !aligned16(d_X) || !aligned16(d_G) || !aligned16(d_dW_rel) ||
      !aligned16(d_dW_root))
    return HIFUSE_ERR_ALIGNMENT;
  if (ws_bytes < hifuse_project_aggregated_bwd_ws_bytes(shape, K, D) || !d_ws)
    return HIFUSE_ERR_WORKSPACE;
  cudaStream_t s = st(stream);
  ProjMeta pm;
  make_proj_meta(m, d_dW_root != nullptr, &pm);
  const int CH = direct_chunk_rows(m);
  float* partial = (float*)d_ws;
  wgrad_tc_launch(m, pm, K, D, CH, nullptr, csr->rel_row_off, nullptr, d_gather_ids,
                  d_X ? d_X : d_Xagg, nullptr, d_G, partial,
                  (unsigned)direct_max_chunks(m, CH), s, d_Xagg);
  int G = d_dW_root ? m.R + m.T : m.R;
  HF_LAUNCH(k_wgrad_reduce, ceil_div((long long)G * K * D / 4, 256), 256, 0, s, m.R, m.T, K * D,
            (const int*)nullptr, (const float4*)partial, (float4*)d_dW_rel, (float4*)d_dW_root,
            pm, csr->rel_row_off, CH, (const float*)nullptr, (const float*)nullptr, 0, 1);
  return last_cuda();
}

hifuse_status hifuse_project_bwd(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                 hifuse_layout layout, hifuse_prec prec, int K, int D, int heads,
                                 const float* d_X, int64_t x_rows, const int32_t* d_gather_ids,
                                 const float* d_W_rel, const float* d_W_root, const float* d_att,
                                 const float* d_Y, float* d_dY, const float* d_G,
                                 const float* d_ds_src, const float* d_ds_dst, float* d_dX,
                                 float* d_dW_rel, float* d_dW_root, float* d_datt, void* d_ws,
                                 size_t ws_bytes, hifuse_stream_t stream) {
  return project_bwd_impl(shape, csr, layout, prec, K, D, heads, d_X, x_rows, d_gather_ids,
                          d_W_rel, d_W_root, d_att, d_Y, d_dY, d_G, d_ds_src, d_ds_dst, d_dX,
                          d_dW_rel, d_dW_root, d_datt, d_ws, ws_bytes, stream, false);
}

hifuse_status hifuse_project_bwd_scored(const hifuse_layer_shape* shape, const hifuse_csr* csr,
                                        hifuse_layout layout, hifuse_prec prec, int K, int D,
                                        int heads, const float* d_X, int64_t x_rows,
                                        const int32_t* d_gather_ids, const float* d_W_rel,
                                        const float* d_W_root, const float* d_att,
                                        const float* d_Y, float* d_dY, const float* d_G,
                                        const float* d_ds_src, const float* d_ds_dst,
                                        float* d_dX, float* d_dW_rel, float* d_dW_root,
                                        float* d_datt, void* d_ws, size_t ws_bytes,
                                        hifuse_stream_t stream) {
  if (!d_att) return HIFUSE_ERR_INVALID_ARG;
  return project_bwd_impl(shape, csr, layout, prec, K, D, heads, d_X, x_rows, d_gather_ids,
                          d_W_rel, d_W_root, d_att, d_Y, d_dY, d_G, d_ds_src, d_ds_dst, d_dX,
                          d_dW_rel, d_dW_root, d_datt, d_ws, ws_bytes, stream, true);
}

}  // extern "C"

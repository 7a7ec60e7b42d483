// head.cu -- training-step helpers outside the paper's four HGNN stages:
// the linear classifier with mean softmax cross-entropy on the seed rows
// (closes the loop of PAPER.md line 156 "forward ... backward
// ... parameter update") and the SGD update.  Deterministic fixed-order sums.
//
// Three kernels for the classifier (deterministic, fixed-order sums):
//  k_head_logits  logits = Hs Wc + bc          (64x64 SIMT tiles)
//  k_head_softmax warp per seed row: dlog = (softmax - onehot) / B, row loss;
//                 the last block sums the per-block losses -> mean loss
//  k_head_grads   one grid, two jobs: dHs = dlog Wc^T and dWc = Hs^T dlog
//                 (+ dbc = column sums of dlog), both split over K with one
//                 partial per slice; the last slice of a tile to finish
//                 (atomic ticket) sums the partials in slice order.
#include <algorithm>
#include "common.cuh"

namespace hf {

static constexpr int kBK = 32;

// One 64x64 tile of C = op(A) op(B) over k in [kb0, kb1): TA: A stored [K][M]
// (else [M][K]); TB: B stored [N][K] (else [K][N]).  256 threads, 4x4 outputs
// each (rows ty + 16i, cols tx + 16j), the next K slab prefetched into
// registers while the current one is used.  colsum: also sum_k B[k][n] for
// this thread's columns (used for dbc), valid in threads with ty == 0.
template <bool TA, bool TB>
__device__ __forceinline__ void gemm_tile(int M, int N, const float* __restrict__ A, int lda,
                                          const float* __restrict__ B, int ldb, int m0, int n0,
                                          int kb0, int kb1, float (&acc)[4][4], bool colsum,
                                          float (&bsum)[4]) {
  __shared__ float As[kBK][64 + 1];
  __shared__ float Bs[kBK][64 + 1];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    bsum[i] = 0.f;
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0.f;
  }
  float ra[8], rb[8];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int i = tid + 256 * q;
      const int kk = TA ? i / 64 : i % kBK, mm = TA ? i % 64 : i / kBK;
      const int m = m0 + mm, k = k0 + kk;
      ra[q] = (m < M && k < kb1) ? (TA ? A[(long long)k * lda + m] : A[(long long)m * lda + k]) : 0.f;
      const int kb = TB ? i % kBK : i / 64, nb = TB ? i / kBK : i % 64;
      const int n = n0 + nb, k2 = k0 + kb;
      rb[q] = (n < N && k2 < kb1) ? (TB ? B[(long long)n * ldb + k2] : B[(long long)k2 * ldb + n]) : 0.f;
    }
  };
  if (kb0 < kb1) fetch(kb0);
  for (int k0 = kb0; k0 < kb1; k0 += kBK) {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int i = tid + 256 * q;
      As[TA ? i / 64 : i % kBK][TA ? i % 64 : i / kBK] = ra[q];
      Bs[TB ? i % kBK : i / 64][TB ? i / kBK : i % 64] = rb[q];
    }
    __syncthreads();
    if (k0 + kBK < kb1) fetch(k0 + kBK);
#pragma unroll
    for (int kk = 0; kk < kBK; kk++) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; i++) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; j++) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      if (colsum) {
#pragma unroll
        for (int j = 0; j < 4; j++) bsum[j] += b[j];
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256)
k_head_logits(int B, int D, int C, const float* __restrict__ Hs, const float* __restrict__ Wc,
              const float* __restrict__ bc, float* __restrict__ lg, int* __restrict__ tickets,
              int ntickets) {
  if (blockIdx.x == 0 && blockIdx.y == 0)   // tickets of the next two kernels
    for (int i = threadIdx.x; i < ntickets; i += blockDim.x) tickets[i] = 0;
  float acc[4][4], bs[4];
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  gemm_tile<false, false>(B, C, Hs, D, Wc, C, m0, n0, 0, D, acc, false, bs);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int n = n0 + tx + 16 * j;
    if (n >= C) continue;
    const float bv = __ldg(bc + n);
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int m = m0 + ty + 16 * i;
      if (m < B) lg[(long long)m * C + n] = acc[i][j] + bv;
    }
  }
}

// 8 rows (one per warp) per block; lg is turned into dlog in place.
__global__ void __launch_bounds__(256)
k_head_softmax(int B, int C, const int* __restrict__ labels, float* __restrict__ lg,
               float* __restrict__ block_loss, int* __restrict__ ticket, float* __restrict__ loss) {
  __shared__ float s_l[8];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = blockIdx.x * 8 + w;
  float rl = 0.f;
  if (b < B) {
    float* x = lg + (long long)b * C;
    float mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = fmaxf(mx, x[c]);
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.f;
    for (int c = lane; c < C; c += 32) se += expf(x[c] - mx);
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const int y = labels[b];
    const float ly = x[y];
    __syncwarp();
    const float inv = 1.f / (float)B;
    for (int c = lane; c < C; c += 32) x[c] = (expf(x[c] - mx) / se - (c == y ? 1.f : 0.f)) * inv;
    rl = logf(se) + mx - ly;
  }
  if (lane == 0) s_l[w] = rl;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int q = 0; q < 8; q++) t += s_l[q];
    block_loss[blockIdx.x] = t;
    __threadfence();
    s_last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    float t = 0.f;
    for (int q = threadIdx.x; q < (int)gridDim.x; q += 32) t += __ldcg(block_loss + q);
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) loss[0] = t / (float)B;
  }
}

struct HeadGrid {
  int dh_tiles_n, dh_tiles, dh_split;       // dHs: [B, D] tiles (n-major), K = C
  int dw_tiles_n, dw_tiles, dw_split;       // dWc: [D, C] tiles, K = B
};

// Sum of the nz slice partials of one 64x64 tile, in slice order, by the last
// slice block to finish.  Returns false in the other blocks.
__device__ __forceinline__ bool last_slice(int* ticket, int nz) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1) == nz - 1;
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

__global__ void __launch_bounds__(256)
k_head_grads(int B, int D, int C, HeadGrid hg, const float* __restrict__ Hs,
             const float* __restrict__ Wc, const float* __restrict__ dlog,
             float* __restrict__ part_h, float* __restrict__ part_w, float* __restrict__ part_b,
             int* __restrict__ tickets, float* __restrict__ dHs, float* __restrict__ dWc,
             float* __restrict__ dbc) {
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4], bs[4];
  int bid = blockIdx.x;
  const int nh = hg.dh_tiles * hg.dh_split;
  if (bid < nh) {
    // ---- dHs = dlog Wc^T: M = B, N = D, K = C; Wc stored [D][C] = [N][K]
    const int tile = bid / hg.dh_split, z = bid % hg.dh_split;
    const int m0 = (tile / hg.dh_tiles_n) * 64, n0 = (tile % hg.dh_tiles_n) * 64;
    const int kper = (C + hg.dh_split - 1) / hg.dh_split;
    gemm_tile<false, true>(B, D, dlog, C, Wc, C, m0, n0, z * kper, min(C, (z + 1) * kper), acc,
                           false, bs);
    float* P = part_h + (long long)z * B * D;
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
        if (m < B && n < D) P[(long long)m * D + n] = acc[i][j];
      }
    if (!last_slice(&tickets[tile], hg.dh_split)) return;
    // all slices' values of a row of 4 outputs in flight together
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int m = m0 + ty + 16 * i;
      float v[4][4];
#pragma unroll
      for (int zz = 0; zz < 4; zz++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int n = n0 + tx + 16 * j;
          v[zz][j] = (zz < hg.dh_split && m < B && n < D)
                         ? __ldcg(part_h + (long long)zz * B * D + (long long)m * D + n) : 0.f;
        }
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int n = n0 + tx + 16 * j;
        float t = v[0][j];
#pragma unroll
        for (int zz = 1; zz < 4; zz++) t += v[zz][j];
        if (m < B && n < D) dHs[(long long)m * D + n] = t;
      }
    }
    return;
  }
  // ---- dWc = Hs^T dlog: M = D, N = C, K = B; Hs stored [B][D] = [K][M]
  bid -= nh;
  const int tile = bid / hg.dw_split, z = bid % hg.dw_split;
  const int m0 = (tile / hg.dw_tiles_n) * 64, n0 = (tile % hg.dw_tiles_n) * 64;
  const int kper = ((B + hg.dw_split - 1) / hg.dw_split + kBK - 1) / kBK * kBK;
  const bool bias = m0 == 0;            // the first row tile also forms dbc
  gemm_tile<true, false>(D, C, Hs, D, dlog, C, m0, n0, z * kper, min(B, (z + 1) * kper), acc,
                         bias, bs);
  float* P = part_w + (long long)z * D * C;
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < D && n < C) P[(long long)m * C + n] = acc[i][j];
    }
  if (bias && ty == 0)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int n = n0 + tx + 16 * j;
      if (n < C) part_b[(long long)z * C + n] = bs[j];
    }
  if (!last_slice(&tickets[hg.dh_tiles + tile], hg.dw_split)) return;
  // 4 outputs x 8 slices in flight per round, summed in slice order
  for (int i = 0; i < 4; i++) {
    const int m = m0 + ty + 16 * i;
    float t[4] = {0.f, 0.f, 0.f, 0.f};
    for (int z0 = 0; z0 < hg.dw_split; z0 += 8) {
      float v[8][4];
#pragma unroll
      for (int u = 0; u < 8; u++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int n = n0 + tx + 16 * j;
          v[u][j] = (z0 + u < hg.dw_split && m < D && n < C)
                        ? __ldcg(part_w + (long long)(z0 + u) * D * C + (long long)m * C + n) : 0.f;
        }
#pragma unroll
      for (int u = 0; u < 8; u++)
#pragma unroll
        for (int j = 0; j < 4; j++) t[j] += v[u][j];
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int n = n0 + tx + 16 * j;
      if (m < D && n < C) dWc[(long long)m * C + n] = t[j];
    }
  }
  if (bias && ty == 0)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int n = n0 + tx + 16 * j;
      if (n >= C) continue;
      float t = 0.f;
      for (int zz = 0; zz < hg.dw_split; zz++) t += __ldcg(part_b + (long long)zz * C + n);
      dbc[n] = t;
    }
}

static HeadGrid head_grid(int B, int D, int C) {
  HeadGrid h;
  h.dh_tiles_n = (int)ceil_div(D, 64);
  h.dh_tiles = h.dh_tiles_n * (int)ceil_div(B, 64);
  h.dh_split = (int)std::max<long long>(1, std::min<long long>(ceil_div(C, 128), 4));   // <= 4
  h.dw_tiles_n = (int)ceil_div(C, 64);
  h.dw_tiles = h.dw_tiles_n * (int)ceil_div(D, 64);
  h.dw_split = (int)std::max<long long>(1, std::min<long long>(ceil_div(B, 128), 32));
  return h;
}

__global__ void k_sgd(float4* __restrict__ p, const float4* __restrict__ g, long long n4, float lr) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  float4 a = p[i], b = g[i];
  a.x -= lr * b.x; a.y -= lr * b.y; a.z -= lr * b.z; a.w -= lr * b.w;
  p[i] = a;
}

__global__ void k_sgd_tail(float* __restrict__ p, const float* __restrict__ g, long long from,
                           long long n, float lr) {
  long long i = from + threadIdx.x;
  if (i < n) p[i] -= lr * g[i];
}

}  // namespace hf

using namespace hf;

extern "C" {

size_t hifuse_xent_ws_bytes(int B, int D, int C) {
  if (B <= 0 || D <= 0 || C <= 0) return 0;
  const HeadGrid h = head_grid(B, D, C);
  const long long nblk = ceil_div(B, 8);
  return carve_bytes((long long)B * C, 4) + carve_bytes(nblk, 4) +
         carve_bytes((long long)h.dh_split * B * D, 4) +
         carve_bytes((long long)h.dw_split * D * C, 4) + carve_bytes((long long)h.dw_split * C, 4) +
         carve_bytes(h.dh_tiles + h.dw_tiles + 1, 4);
}

hifuse_status hifuse_linear_xent(int B, int D, int C, const float* d_H, int64_t h_rows,
                                 int64_t h_row0, const int32_t* d_labels, const float* d_Wc,
                                 const float* d_bc, float* d_loss, float* d_dH, float* d_dWc,
                                 float* d_dbc, void* d_ws, size_t ws_bytes,
                                 hifuse_stream_t stream) {
  if (B <= 0 || D <= 0 || C <= 0 || h_row0 < 0 || h_row0 + B > h_rows || !d_H || !d_labels ||
      !d_Wc || !d_bc || !d_loss || !d_dH || !d_dWc || !d_dbc)
    return HIFUSE_ERR_INVALID_ARG;
  if (ws_bytes < hifuse_xent_ws_bytes(B, D, C) || !d_ws) return HIFUSE_ERR_WORKSPACE;
  cudaStream_t s = st(stream);
  const HeadGrid h = head_grid(B, D, C);
  const int nblk = (int)ceil_div(B, 8);
  char* p = (char*)d_ws;
  float* dlog = carve<float>(p, (long long)B * C);
  float* block_loss = carve<float>(p, nblk);
  float* part_h = carve<float>(p, (long long)h.dh_split * B * D);
  float* part_w = carve<float>(p, (long long)h.dw_split * D * C);
  float* part_b = carve<float>(p, (long long)h.dw_split * C);
  int* tickets = carve<int>(p, h.dh_tiles + h.dw_tiles + 1);
  const int ntk = h.dh_tiles + h.dw_tiles + 1;       // last one: the softmax ticket
  // rows of dH outside the seeds get no gradient
  if (h_row0 > 0) cudaMemsetAsync(d_dH, 0, sizeof(float) * h_row0 * D, s);
  if (h_row0 + B < h_rows)
    cudaMemsetAsync(d_dH + (h_row0 + B) * D, 0, sizeof(float) * (h_rows - h_row0 - B) * D, s);
  const float* Hs = d_H + h_row0 * D;
  HF_LAUNCH(k_head_logits, dim3(ceil_div(C, 64), ceil_div(B, 64)), 256, 0, s, B, D, C, Hs, d_Wc,
            d_bc, dlog, tickets, ntk);
  HF_LAUNCH(k_head_softmax, nblk, 256, 0, s, B, C, d_labels, dlog, block_loss, tickets + ntk - 1,
            d_loss);
  HF_LAUNCH(k_head_grads, h.dh_tiles * h.dh_split + h.dw_tiles * h.dw_split, 256, 0, s, B, D, C,
            h, Hs, d_Wc, dlog, part_h, part_w, part_b, tickets, d_dH + h_row0 * D, d_dWc, d_dbc);
  return last_cuda();
}

hifuse_status hifuse_sgd(float* d_param, const float* d_grad, int64_t n, float lr,
                         float grad_scale, hifuse_stream_t stream) {
  if (n < 0 || (n > 0 && (!d_param || !d_grad))) return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_param) || !aligned16(d_grad)) return HIFUSE_ERR_ALIGNMENT;
  cudaStream_t s = st(stream);
  long long n4 = n / 4;
  float a = lr * grad_scale;
  HF_LAUNCH(k_sgd, ceil_div(n4, 256), 256, 0, s, (float4*)d_param, (const float4*)d_grad, n4, a);
  if (n4 * 4 < n) HF_LAUNCH(k_sgd_tail, 1, 32, 0, s, d_param, d_grad, n4 * 4, (long long)n, a);
  return last_cuda();
}

}  // extern "C"

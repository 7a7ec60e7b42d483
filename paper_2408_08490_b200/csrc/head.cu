// head.cu -- training-step helpers outside the paper's four HGNN stages:
// the linear classifier with mean softmax cross-entropy on the seed rows
// (closes the loop of PAPER.md line 156 "forward ... backward
// ... parameter update") and the SGD update.  Deterministic fixed-order sums.
#include "common.cuh"

namespace hf {

static constexpr int kSplit = 16;

__device__ __forceinline__ float block_reduce(float v, float* sm, bool is_max) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = 16; o; o >>= 1) {
    float n = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, n) : v + n;
  }
  __syncthreads();
  if (lane == 0) sm[w] = v;
  __syncthreads();
  float r = sm[0];
  for (int i = 1; i < nw; i++) r = is_max ? fmaxf(r, sm[i]) : r + sm[i];
  return r;
}

// Small SIMT GEMM: C[M,N] = op(A)[M,K] op(B)[K,N]; TA: A stored [K,M]; TB: B
// stored [N,K].  64x64 tiles, 256 threads, 4x4 outputs per thread, BK = 32,
// the next K tile prefetched into registers while the current one is used.
// gridDim.z > 1: split-K, slice z writes C + z*M*ldc (summed in fixed order).
template <bool TA, bool TB>
__global__ void __launch_bounds__(256)
k_gemm_small(int M, int N, int K, const float* __restrict__ A, int lda,
             const float* __restrict__ B, int ldb, float* __restrict__ C, int ldc,
             long long a_row0, long long c_row0) {
  constexpr int BK = 32;
  __shared__ float As[BK][64 + 1];
  __shared__ float Bs[BK][64 + 1];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int kper = ((K + gridDim.z - 1) / gridDim.z + BK - 1) / BK * BK;
  const int kb0 = blockIdx.z * kper, kb1 = min(K, kb0 + kper);
  C += (long long)blockIdx.z * M * ldc;
  float acc[4][4] = {};
  float ra[8], rb[8];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int i = tid + 256 * q;
      int kk = TA ? i / 64 : i % BK, mm = TA ? i % 64 : i / BK;
      int m = m0 + mm, k = k0 + kk;
      ra[q] = (m < M && k < kb1) ? (TA ? A[(long long)k * lda + a_row0 + m] : A[(a_row0 + m) * lda + k]) : 0.f;
      int kb = TB ? i % BK : i / 64, nb = TB ? i / BK : i % 64;
      int n = n0 + nb, k2 = k0 + kb;
      rb[q] = (n < N && k2 < kb1) ? (TB ? B[(long long)n * ldb + k2] : B[(long long)k2 * ldb + n]) : 0.f;
    }
  };
  if (kb0 < kb1) fetch(kb0);
  for (int k0 = kb0; k0 < kb1; k0 += BK) {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int i = tid + 256 * q;
      As[TA ? i / 64 : i % BK][TA ? i % 64 : i / BK] = ra[q];
      Bs[TB ? i % BK : i / 64][TB ? i / BK : i % 64] = rb[q];
    }
    __syncthreads();
    if (k0 + BK < kb1) fetch(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk++) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; i++) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; j++) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      int n = n0 + tx + 16 * j;
      if (n < N) C[(c_row0 + m) * ldc + n] = acc[i][j];
    }
  }
}

// One warp per seed row: bias, softmax over the C logits (in place ->
// dlogits = (softmax - onehot) / B), per-row loss.
__global__ void k_xent_softmax(int B, int C, const float* __restrict__ bc,
                               const int* __restrict__ labels, float* __restrict__ lg,
                               float* __restrict__ row_loss) {
  int b = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (b >= B) return;
  float* x = lg + (long long)b * C;
  float mx = -INFINITY;
  for (int c = lane; c < C; c += 32) {
    float v = x[c] + bc[c];
    x[c] = v;
    mx = fmaxf(mx, v);
  }
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float se = 0.f;
  for (int c = lane; c < C; c += 32) se += expf(x[c] - mx);
  for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  int y = labels[b];
  __syncwarp();
  float ly = x[y];
  __syncwarp();
  float inv = 1.f / (float)B;
  for (int c = lane; c < C; c += 32) x[c] = (expf(x[c] - mx) / se - (c == y ? 1.f : 0.f)) * inv;
  if (lane == 0) row_loss[b] = logf(se) + mx - ly;
}

__global__ void k_xent_loss(int B, const float* __restrict__ row_loss, float* __restrict__ loss) {
  __shared__ float red[32];
  float s = 0.f;
  for (int b = threadIdx.x; b < B; b += blockDim.x) s += row_loss[b];
  s = block_reduce(s, red, false);
  if (threadIdx.x == 0) loss[0] = s / (float)B;
}

// dbc[c] = sum_b dlog[b][c]: 32 columns x 8 row groups per block, fixed-order
// shared-memory combine (deterministic).
__global__ void __launch_bounds__(256)
k_xent_dbias(int B, int C, const float* __restrict__ dlog, float* __restrict__ dbc) {
  __shared__ float red[8][33];
  int c = blockIdx.x * 32 + (threadIdx.x & 31), g = threadIdx.x >> 5;
  float s = 0.f;
  if (c < C)
    for (int b = g; b < B; b += 8) s += dlog[(long long)b * C + c];
  red[g][threadIdx.x & 31] = s;
  __syncthreads();
  if (g == 0 && c < C) {
    float t = red[0][threadIdx.x];
    for (int q = 1; q < 8; q++) t += red[q][threadIdx.x];
    dbc[c] = t;
  }
}

// sum of split-K partials, fixed order
__global__ void k_sum_splits(int n, int splits, const float* __restrict__ part,
                             float* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int z = 0; z < splits; z++) s += part[(long long)z * n + i];
  out[i] = s;
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
  (void)D;
  long long np = (long long)kSplit * D * C;
  if (np < 4ll * B * D) np = 4ll * B * D;
  if (np < 4ll * B * C) np = 4ll * B * C;
  return carve_bytes((long long)B * C, 4) + carve_bytes(B, 4) + carve_bytes(np, 4);
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
  char* p = (char*)d_ws;
  float* dlog = carve<float>(p, (long long)B * C);
  float* row_loss = carve<float>(p, B);
  long long np = (long long)kSplit * D * C;
  if (np < 4ll * B * D) np = 4ll * B * D;
  if (np < 4ll * B * C) np = 4ll * B * C;
  float* part = carve<float>(p, np);
  cudaMemsetAsync(d_dH, 0, sizeof(float) * h_rows * D, s);
  // logits = Hs Wc  (split-K 4, fixed-order sum)
  dim3 g1(ceil_div(C, 64), ceil_div(B, 64), 4);
  HF_LAUNCH((k_gemm_small<false, false>), g1, 256, 0, s, B, C, D, d_H, D, d_Wc, C, part, C,
            (long long)h_row0, 0ll);
  HF_LAUNCH(k_sum_splits, ceil_div((long long)B * C, 256), 256, 0, s, B * C, 4, part, dlog);
  HF_LAUNCH(k_xent_softmax, ceil_div(B, 8), 256, 0, s, B, C, d_bc, d_labels, dlog, row_loss);
  HF_LAUNCH(k_xent_loss, 1, 256, 0, s, B, row_loss, d_loss);
  // dHs = dlog Wc^T   (Wc is [D, C]: op(B) = Wc^T stored [N = D, K = C])
  dim3 g2(ceil_div(D, 64), ceil_div(B, 64), 4);
  HF_LAUNCH((k_gemm_small<false, true>), g2, 256, 0, s, B, D, C, dlog, C, d_Wc, C, part, D, 0ll,
            0ll);
  HF_LAUNCH(k_sum_splits, ceil_div((long long)B * D, 256), 256, 0, s, B * D, 4, part,
            d_dH + h_row0 * D);
  // dWc = Hs^T dlog: split-K over the batch, then a fixed-order sum
  dim3 g3(ceil_div(C, 64), ceil_div(D, 64), kSplit);
  HF_LAUNCH((k_gemm_small<true, false>), g3, 256, 0, s, D, C, B, d_H + h_row0 * D, D, dlog, C,
            part, C, 0ll, 0ll);
  HF_LAUNCH(k_sum_splits, ceil_div((long long)D * C, 256), 256, 0, s, D * C, kSplit, part, d_dWc);
  HF_LAUNCH(k_xent_dbias, ceil_div(C, 32), 256, 0, s, B, C, dlog, d_dbc);
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

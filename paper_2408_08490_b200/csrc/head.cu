// head.cu -- training-step helpers outside the paper's four HGNN stages:
// the linear classifier with mean softmax cross-entropy on the seed rows
// (closes the loop of PAPER.md line 156 "forward ... backward
// ... parameter update") and the SGD update.  Deterministic fixed-order sums.
#include "common.cuh"

namespace hf {

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

// one block per seed row: logits, softmax, per-row loss and dlogits
__global__ void k_xent_rows(int B, int D, int C, const float* __restrict__ H, long long h_row0,
                            const int* __restrict__ labels, const float* __restrict__ Wc,
                            const float* __restrict__ bc, float* __restrict__ dlog,
                            float* __restrict__ row_loss) {
  extern __shared__ float sm[];   // [D] h row, [C] logits, [32] scratch
  float* hrow = sm;
  float* lg = sm + D;
  float* red = lg + C;
  int b = blockIdx.x;
  for (int d = threadIdx.x; d < D; d += blockDim.x) hrow[d] = H[(h_row0 + b) * D + d];
  __syncthreads();
  float mx = -INFINITY;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s = bc[c];
    for (int d = 0; d < D; d++) s = fmaf(hrow[d], Wc[(long long)d * C + c], s);
    lg[c] = s;
    mx = fmaxf(mx, s);
  }
  mx = block_reduce(mx, red, true);
  float se = 0.f;
  for (int c = threadIdx.x; c < C; c += blockDim.x) se += expf(lg[c] - mx);
  se = block_reduce(se, red, false);
  int y = labels[b];
  float inv = 1.f / (float)B;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float p = expf(lg[c] - mx) / se;
    dlog[(long long)b * C + c] = (p - (c == y ? 1.f : 0.f)) * inv;
  }
  if (threadIdx.x == 0) row_loss[b] = logf(se) + mx - lg[y];
}

__global__ void k_xent_loss(int B, const float* __restrict__ row_loss, float* __restrict__ loss) {
  __shared__ float red[32];
  float s = 0.f;
  for (int b = threadIdx.x; b < B; b += blockDim.x) s += row_loss[b];
  s = block_reduce(s, red, false);
  if (threadIdx.x == 0) loss[0] = s / (float)B;
}

// dH[h_row0 + b][d] = sum_c dlog[b][c] Wc[d][c]
__global__ void k_xent_dh(int B, int D, int C, long long h_row0, const float* __restrict__ dlog,
                          const float* __restrict__ Wc, float* __restrict__ dH) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)B * D) return;
  int b = (int)(idx / D), d = (int)(idx % D);
  float s = 0.f;
  for (int c = 0; c < C; c++) s = fmaf(dlog[(long long)b * C + c], Wc[(long long)d * C + c], s);
  dH[(h_row0 + b) * D + d] = s;
}

// dWc[d][c] = sum_b H[b][d] dlog[b][c];  dbc[c] = sum_b dlog[b][c]
__global__ void k_xent_dw(int B, int D, int C, long long h_row0, const float* __restrict__ H,
                          const float* __restrict__ dlog, float* __restrict__ dWc,
                          float* __restrict__ dbc) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)(D + 1) * C) return;
  int d = (int)(idx / C), c = (int)(idx % C);
  float s = 0.f;
  if (d < D) {
    for (int b = 0; b < B; b++) s = fmaf(H[(h_row0 + b) * D + d], dlog[(long long)b * C + c], s);
    dWc[(long long)d * C + c] = s;
  } else {
    for (int b = 0; b < B; b++) s += dlog[(long long)b * C + c];
    dbc[c] = s;
  }
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
  return carve_bytes((long long)B * C, 4) + carve_bytes(B, 4);
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
  size_t smem = (size_t)(D + C + 32) * sizeof(float);
  if (smem > 48 * 1024) return HIFUSE_ERR_UNSUPPORTED;
  cudaStream_t s = st(stream);
  char* p = (char*)d_ws;
  float* dlog = carve<float>(p, (long long)B * C);
  float* row_loss = carve<float>(p, B);
  cudaMemsetAsync(d_dH, 0, sizeof(float) * h_rows * D, s);
  HF_LAUNCH(k_xent_rows, B, 128, smem, s, B, D, C, d_H, (long long)h_row0, d_labels, d_Wc, d_bc,
            dlog, row_loss);
  HF_LAUNCH(k_xent_loss, 1, 256, 0, s, B, row_loss, d_loss);
  HF_LAUNCH(k_xent_dh, ceil_div((long long)B * D, 256), 256, 0, s, B, D, C, (long long)h_row0,
            dlog, d_Wc, d_dH);
  HF_LAUNCH(k_xent_dw, ceil_div((long long)(D + 1) * C, 256), 256, 0, s, B, D, C,
            (long long)h_row0, d_H, dlog, d_dWc, d_dbc);
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

// fuse.cu -- A5 semantic fusion ("integrates semantic
// information across all semantic graphs by combining the results") and its
// backward.  Readings C2/C4/C10: H_t[i] = act(R0_t[i] + b_t + sum_{r: t(r)=t}
// Z[rel_row_off[r] + i]); ReLU between layers, none after the last.
#include "common.cuh"

namespace hf {

struct FuseMeta {
  int T, D4, dst_rows;
  int type_dst_off[HF_MAX_T + 1];
  int list_off[HF_MAX_T + 1];      // relations into type t: rel_rows[list_off[t]..list_off[t+1])
  int rel_rows[HF_MAX_R];          // rel_row_off of each listed relation
};

static void make_fuse_meta(const LayerMeta& m, int D, FuseMeta* f) {
  f->T = m.T;
  f->D4 = D / 4;
  f->dst_rows = m.dst_rows;
  int k = 0;
  for (int t = 0; t <= m.T; t++) f->type_dst_off[t] = m.type_dst_off[t];
  for (int t = 0; t < m.T; t++) {
    f->list_off[t] = k;
    for (int r = 0; r < m.R; r++)
      if (m.rel_dst[r] == t) f->rel_rows[k++] = m.rel_row_off[r];
  }
  f->list_off[m.T] = k;
}

template <bool RELU>
__global__ void k_fuse(FuseMeta f, const float4* __restrict__ Z, const float4* __restrict__ R0,
                       const float4* __restrict__ bias, float4* __restrict__ H) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)f.dst_rows * f.D4) return;
  int o = (int)(idx / f.D4), c = (int)(idx % f.D4);
  int t = upper_bound_i(f.type_dst_off, f.T + 1, o) - 1;
  int i = o - f.type_dst_off[t];
  float4 v = R0 ? R0[idx] : make_float4(0.f, 0.f, 0.f, 0.f);
  if (bias) {
    float4 b = bias[t * f.D4 + c];
    v.x += b.x; v.y += b.y; v.z += b.z; v.w += b.w;
  }
  for (int k = f.list_off[t]; k < f.list_off[t + 1]; k++) {
    float4 z = __ldg(Z + (long long)(f.rel_rows[k] + i) * f.D4 + c);
    v.x += z.x; v.y += z.y; v.z += z.z; v.w += z.w;
  }
  if (RELU) {
    v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
  }
  H[idx] = v;
}

// Backward stage 1: chunk c (kChunk rows of one type) writes G = dH * act'(H)
// and the chunk's column sums; stage 2 sums a type's chunks in order.
static constexpr int kChunk = 64;

struct FuseBwdMeta {
  int T, D4;
  int type_dst_off[HF_MAX_T + 1];
  int chunk_off[HF_MAX_T + 1];
};

template <bool RELU>
__global__ void __launch_bounds__(256)
k_fuse_bwd_chunks(FuseBwdMeta f, const float4* __restrict__ dH, const float4* __restrict__ Hv,
                  float4* __restrict__ G, float4* __restrict__ partial) {
  __shared__ float4 red[256];
  int c = blockIdx.x;
  int t = upper_bound_i(f.chunk_off, f.T + 1, c) - 1;
  int row0 = f.type_dst_off[t] + (c - f.chunk_off[t]) * kChunk;
  int row1 = min(row0 + kChunk, f.type_dst_off[t + 1]);
  int col = threadIdx.x % f.D4, sub = threadIdx.x / f.D4, nsub = 256 / f.D4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int o = row0 + sub; o < row1; o += nsub) {
    long long idx = (long long)o * f.D4 + col;
    float4 g = dH[idx];
    if (RELU) {
      float4 h = Hv[idx];
      g.x = h.x > 0.f ? g.x : 0.f; g.y = h.y > 0.f ? g.y : 0.f;
      g.z = h.z > 0.f ? g.z : 0.f; g.w = h.w > 0.f ? g.w : 0.f;
    }
    G[idx] = g;
    acc.x += g.x; acc.y += g.y; acc.z += g.z; acc.w += g.w;
  }
  if (!partial) return;
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < f.D4) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < nsub; k++) {
      float4 v = red[k * f.D4 + threadIdx.x];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    partial[(long long)c * f.D4 + threadIdx.x] = s;
  }
}

// one block per type: threads split the type's chunks, fixed-order smem reduce
__global__ void __launch_bounds__(256)
k_fuse_bwd_bias(FuseBwdMeta f, const float4* __restrict__ partial, float4* __restrict__ dbias) {
  __shared__ float4 red[256];
  int t = blockIdx.x;
  int c = threadIdx.x % f.D4, sub = threadIdx.x / f.D4, nsub = 256 / f.D4;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = f.chunk_off[t] + sub; k < f.chunk_off[t + 1]; k += nsub) {
    float4 v = partial[(long long)k * f.D4 + c];
    s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < f.D4) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < nsub; k++) {
      float4 v = red[k * f.D4 + threadIdx.x];
      a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
    }
    dbias[t * f.D4 + threadIdx.x] = a;
  }
}

static void make_fbm(const LayerMeta& m, int D, FuseBwdMeta* f) {
  f->T = m.T;
  f->D4 = D / 4;
  int k = 0;
  for (int t = 0; t <= m.T; t++) f->type_dst_off[t] = m.type_dst_off[t];
  for (int t = 0; t < m.T; t++) {
    f->chunk_off[t] = k;
    k += (m.n_dst[t] + kChunk - 1) / kChunk;
  }
  f->chunk_off[m.T] = k;
}

}  // namespace hf

using namespace hf;

extern "C" {

hifuse_status hifuse_semantic_fuse(const hifuse_layer_shape* shape, int D, hifuse_act act,
                                   const float* d_Z, const float* d_R0, const float* d_bias,
                                   float* d_H, hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (D != 64 && D != 128) return HIFUSE_ERR_UNSUPPORTED;
  if (m.dst_rows > 0 && (!d_H || (!d_Z && m.rows > 0))) return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_Z) || !aligned16(d_R0) || !aligned16(d_bias) || !aligned16(d_H))
    return HIFUSE_ERR_ALIGNMENT;
  FuseMeta f;
  make_fuse_meta(m, D, &f);
  long long n = (long long)m.dst_rows * (D / 4);
  unsigned grid = ceil_div(n, 256);
  cudaStream_t s = st(stream);
  if (act == HIFUSE_ACT_RELU)
    HF_LAUNCH(k_fuse<true>, grid, 256, 0, s, f, (const float4*)d_Z, (const float4*)d_R0,
              (const float4*)d_bias, (float4*)d_H);
  else if (act == HIFUSE_ACT_NONE)
    HF_LAUNCH(k_fuse<false>, grid, 256, 0, s, f, (const float4*)d_Z, (const float4*)d_R0,
              (const float4*)d_bias, (float4*)d_H);
  else
    return HIFUSE_ERR_INVALID_ARG;
  return last_cuda();
}

size_t hifuse_fuse_bwd_ws_bytes(const hifuse_layer_shape* shape, int D) {
  LayerMeta m;
  if (make_meta(shape, &m) != HIFUSE_OK) return 0;
  FuseBwdMeta f;
  make_fbm(m, D, &f);
  return carve_bytes((long long)(f.chunk_off[m.T] + 1) * D, 4);
}

hifuse_status hifuse_semantic_fuse_bwd(const hifuse_layer_shape* shape, int D, hifuse_act act,
                                       const float* d_dH, const float* d_H, float* d_G,
                                       float* d_dbias, void* d_ws, size_t ws_bytes,
                                       hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (D != 64 && D != 128) return HIFUSE_ERR_UNSUPPORTED;
  if (m.dst_rows > 0 && (!d_dH || !d_G || (act == HIFUSE_ACT_RELU && !d_H)))
    return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_dH) || !aligned16(d_H) || !aligned16(d_G) || !aligned16(d_dbias))
    return HIFUSE_ERR_ALIGNMENT;
  if (d_dbias && (ws_bytes < hifuse_fuse_bwd_ws_bytes(shape, D) || !d_ws))
    return HIFUSE_ERR_WORKSPACE;
  FuseBwdMeta f;
  make_fbm(m, D, &f);
  cudaStream_t s = st(stream);
  float4* partial = d_dbias ? (float4*)d_ws : nullptr;
  int nch = f.chunk_off[m.T];
  if (act == HIFUSE_ACT_RELU)
    HF_LAUNCH(k_fuse_bwd_chunks<true>, nch, 256, 0, s, f, (const float4*)d_dH, (const float4*)d_H,
              (float4*)d_G, partial);
  else
    HF_LAUNCH(k_fuse_bwd_chunks<false>, nch, 256, 0, s, f, (const float4*)d_dH,
              (const float4*)d_H, (float4*)d_G, partial);
  if (d_dbias)
    HF_LAUNCH(k_fuse_bwd_bias, m.T, 256, 0, s, f, partial, (float4*)d_dbias);
  return last_cuda();
}

}  // extern "C"

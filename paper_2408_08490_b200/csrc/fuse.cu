// fuse.cu -- A5 semantic fusion ("integrates semantic
// information across all semantic graphs by combining the results") and its
// backward.  Readings C2/C4/C10: H_t[i] = act(R0_t[i] + b_t + sum_{r: t(r)=t}
// Z[rel_row_off[r] + i]); ReLU between layers, none after the last.
#include <algorithm>
#include "common.cuh"

namespace hf {

struct FuseMeta {
  int T, D4, dst_rows;
  int type_dst_off[HF_MAX_T + 1];
  int list_off[HF_MAX_T + 1];      // relations into type t: rel_rows[list_off[t]..list_off[t+1])
  int rel_rows[HF_MAX_R];          // rel_row_off of each listed relation
  int rel_idx[HF_MAX_R];           // its relation id (index into beta)
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
      if (m.rel_dst[r] == t) {
        f->rel_idx[k] = r;
        f->rel_rows[k++] = m.rel_row_off[r];
      }
  }
  f->list_off[m.T] = k;
}

template <bool RELU>
__global__ void k_fuse(FuseMeta f, const float4* __restrict__ Z, const float4* __restrict__ R0,
                       const float4* __restrict__ bias, float4* __restrict__ H,
                       const float* __restrict__ beta) {
  HF_PDL_ENTRY();
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
    if (beta) {                    // HAN semantic-attention weight of the relation
      const float w = __ldg(beta + f.rel_idx[k]);
      v.x = fmaf(w, z.x, v.x); v.y = fmaf(w, z.y, v.y); v.z = fmaf(w, z.z, v.z);
      v.w = fmaf(w, z.w, v.w);
    } else {
      v.x += z.x; v.y += z.y; v.z += z.z; v.w += z.w;
    }
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

// WRITE_G = false: G is an input (dH = G, no ReLU), only the chunk column
// sums are formed (hifuse_semantic_fuse_bwd_bias).
template <bool RELU, bool WRITE_G = true>
__global__ void __launch_bounds__(256)
k_fuse_bwd_chunks(FuseBwdMeta f, const float4* __restrict__ dH, const float4* __restrict__ Hv,
                  float4* __restrict__ G, float4* __restrict__ partial) {
  HF_PDL_ENTRY();
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
    if (WRITE_G) G[idx] = g;
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
  HF_PDL_ENTRY();
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


// ------------------------------------------------- HAN semantic attention --
// SURVEY.md §8(f) NEXT(2), reading C22 (PAPER.md line 123 leaves the fusion
// rule open; HAN's semantic-level attention [ext]):
//   w_r = (1/n_t) sum_i q . tanh(Ws^T Z[(r,i)] + bs),  beta = softmax_r|t(r)=t (w)
//   H_t[i] = act(R0 + b + sum_r beta_r Z[(r,i)])
// Per merged row the A-vector a = Ws^T z + bs is a (D x A) matvec: a warp
// takes kSemRPW rows at once (z rows staged in shared memory, Ws staged once
// per block with row stride A + 1 so that both the lane-over-A (forward) and
// the lane-over-D (dZ = Ws g) accesses are bank-conflict free).  All
// reductions (per relation, per column) have a fixed order.
constexpr int kSemRPW = 8;
constexpr int kSemWarps = 8;

struct SemMeta {
  int R, T, rows;
  int rel_row_off[HF_MAX_R + 1];
  int shift[HF_MAX_R];           // G row of merged row m = m + shift[r(m)]
  int n_t[HF_MAX_R];             // n_dst of the destination type of r
  int rel_dst[HF_MAX_R];
};

static void make_sem_meta(const LayerMeta& m, SemMeta* sm) {
  sm->R = m.R;
  sm->T = m.T;
  sm->rows = m.rows;
  for (int r = 0; r <= m.R; r++) sm->rel_row_off[r] = m.rel_row_off[r];
  for (int r = 0; r < m.R; r++) {
    sm->shift[r] = m.type_dst_off[m.rel_dst[r]] - m.rel_row_off[r];
    sm->n_t[r] = m.n_dst[m.rel_dst[r]];
    sm->rel_dst[r] = m.rel_dst[r];
  }
}

template <int D, int A>
constexpr size_t sem_smem() {
  return sizeof(float) * ((size_t)D * (A + 1) + (size_t)kSemWarps * kSemRPW * (D > A ? D : A));
}

// BWD = false: s_out[m] = q . tanh(Ws^T Z[m] + bs).
// BWD = true : with c_r = coef[r] = dw_r / n_t, ga = c_r q (.) (1 - tanh^2(a)):
//              dZ[m] = beta_r G[m + shift] + Ws ga;  Ga[m] = ga;  Th[m] = c_r tanh(a).
template <int D, int A, bool BWD>
__global__ void __launch_bounds__(kSemWarps * 32)
k_sem_rows(SemMeta sm, const float* __restrict__ Z, const float* __restrict__ Ws,
           const float* __restrict__ bs, const float* __restrict__ q, float* __restrict__ s_out,
           const float* __restrict__ G, const float* __restrict__ beta,
           const float* __restrict__ coef, float* __restrict__ dZ, float* __restrict__ Ga,
           float* __restrict__ Th) {
  HF_PDL_ENTRY();
  constexpr int AP = A + 1, KA = A / 32, KD = D / 32, RW = D > A ? D : A;
  extern __shared__ float ssm[];
  float* sW = ssm;                                  // [D][A+1]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* zs = ssm + D * AP + w * kSemRPW * RW;      // [kSemRPW][RW] per warp
  // stage Ws (8 loads in flight per thread)
  for (int i0 = 0; i0 < D * A; i0 += 8 * blockDim.x) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int i = i0 + k * blockDim.x + threadIdx.x;
      v[k] = i < D * A ? __ldg(Ws + i) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int i = i0 + k * blockDim.x + threadIdx.x;
      if (i < D * A) sW[(i / A) * AP + (i % A)] = v[k];
    }
  }
  __syncthreads();
  float bv[KA], qv[KA];
#pragma unroll
  for (int k = 0; k < KA; k++) {
    bv[k] = __ldg(bs + lane + 32 * k);
    qv[k] = __ldg(q + lane + 32 * k);
  }
  const int nwarps = gridDim.x * kSemWarps;
  for (int m0 = (blockIdx.x * kSemWarps + w) * kSemRPW; m0 < sm.rows; m0 += nwarps * kSemRPW) {
    // stage the rows' z (float4 loads all in flight)
    {
      constexpr int F4 = D / 4;
      float4 v[kSemRPW * F4 / 32 > 0 ? kSemRPW * F4 / 32 : 1];
#pragma unroll
      for (int k = 0; k < kSemRPW * F4 / 32; k++) {
        const int idx = k * 32 + lane, r = idx / F4, c4 = idx % F4;
        v[k] = m0 + r < sm.rows ? __ldg(reinterpret_cast<const float4*>(Z + (long long)(m0 + r) * D) + c4)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < kSemRPW * F4 / 32; k++) {
        const int idx = k * 32 + lane, r = idx / F4, c4 = idx % F4;
        reinterpret_cast<float4*>(zs + r * RW)[c4] = v[k];
      }
    }
    __syncwarp();
    float acc[kSemRPW][KA];
#pragma unroll
    for (int r = 0; r < kSemRPW; r++)
#pragma unroll
      for (int k = 0; k < KA; k++) acc[r][k] = bv[k];
#pragma unroll 4
    for (int d = 0; d < D; d++) {
      float wv[KA];
#pragma unroll
      for (int k = 0; k < KA; k++) wv[k] = sW[d * AP + lane + 32 * k];
#pragma unroll
      for (int r = 0; r < kSemRPW; r++) {
        const float z = zs[r * RW + d];
#pragma unroll
        for (int k = 0; k < KA; k++) acc[r][k] = fmaf(z, wv[k], acc[r][k]);
      }
    }
    if (!BWD) {
#pragma unroll
      for (int r = 0; r < kSemRPW; r++) {
        float sum = 0.f;
#pragma unroll
        for (int k = 0; k < KA; k++) sum = fmaf(qv[k], tanhf(acc[r][k]), sum);
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0 && m0 + r < sm.rows) s_out[m0 + r] = sum;
      }
      continue;
    }
    // backward: ga, Th, and dZ = beta G + Ws ga
    int rel[kSemRPW];
#pragma unroll
    for (int r = 0; r < kSemRPW; r++) {
      const int m = min(m0 + r, sm.rows - 1);
      int lo = 0, hi = sm.R;                         // rel_row_off[lo] <= m < rel_row_off[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (sm.rel_row_off[mid] <= m) lo = mid; else hi = mid;
      }
      rel[r] = lo;
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kSemRPW; r++) {
      const float cf = __ldg(coef + rel[r]);
      const bool in = m0 + r < sm.rows;
#pragma unroll
      for (int k = 0; k < KA; k++) {
        const float th = tanhf(acc[r][k]);
        const float ga = cf * qv[k] * (1.f - th * th);
        zs[r * RW + lane + 32 * k] = ga;            // z no longer needed
        if (in) {
          Ga[(long long)(m0 + r) * A + lane + 32 * k] = ga;
          Th[(long long)(m0 + r) * A + lane + 32 * k] = cf * th;
        }
      }
    }
    __syncwarp();
    float acc2[kSemRPW][KD];
#pragma unroll
    for (int r = 0; r < kSemRPW; r++)
#pragma unroll
      for (int k = 0; k < KD; k++) acc2[r][k] = 0.f;
#pragma unroll 4
    for (int c = 0; c < A; c++) {
      float wv[KD];
#pragma unroll
      for (int k = 0; k < KD; k++) wv[k] = sW[(lane + 32 * k) * AP + c];
#pragma unroll
      for (int r = 0; r < kSemRPW; r++) {
        const float g = zs[r * RW + c];
#pragma unroll
        for (int k = 0; k < KD; k++) acc2[r][k] = fmaf(wv[k], g, acc2[r][k]);
      }
    }
#pragma unroll
    for (int r = 0; r < kSemRPW; r++) {
      const int m = m0 + r;
      if (m >= sm.rows) continue;
      const float bt = __ldg(beta + rel[r]);
      const long long gr = (long long)(m + sm.shift[rel[r]]) * D;
#pragma unroll
      for (int k = 0; k < KD; k++) {
        const int d = lane + 32 * k;
        dZ[(long long)m * D + d] = fmaf(bt, __ldg(G + gr + d), acc2[r][k]);
      }
    }
    __syncwarp();
  }
}

// One block: per relation the fixed-order mean of s over its rows (FWD:
// w_r, then beta = softmax per destination type) or the sum of dd (BWD:
// dbeta_r, then coef_r = beta_r (dbeta_r - sum_{r'|t} beta_r' dbeta_r') / n_t).
template <bool BWD>
__global__ void __launch_bounds__(256)
k_sem_rel(SemMeta sm, const float* __restrict__ s, const float* __restrict__ beta_in,
          float* __restrict__ out, float* __restrict__ w_out) {
  HF_PDL_ENTRY();
  __shared__ float red[256];
  __shared__ float val[HF_MAX_R];
  for (int r = 0; r < sm.R; r++) {
    const int a = sm.rel_row_off[r], n = sm.rel_row_off[r + 1] - a;
    float acc = 0.f;
    for (int i = threadIdx.x; i < n; i += 256) acc += s[a + i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) val[r] = BWD ? red[0] : (n > 0 ? red[0] / (float)n : 0.f);
    __syncthreads();
  }
  for (int r = threadIdx.x; r < sm.R; r += 256) {
    const int t = sm.rel_dst[r];
    if (!BWD) {
      float mx = -INFINITY;
      for (int r2 = 0; r2 < sm.R; r2++) if (sm.rel_dst[r2] == t) mx = fmaxf(mx, val[r2]);
      float sum = 0.f;
      for (int r2 = 0; r2 < sm.R; r2++) if (sm.rel_dst[r2] == t) sum += expf(val[r2] - mx);
      out[r] = expf(val[r] - mx) / sum;
      if (w_out) w_out[r] = val[r];
    } else {
      float sb = 0.f;
      for (int r2 = 0; r2 < sm.R; r2++)
        if (sm.rel_dst[r2] == t) sb = fmaf(beta_in[r2], val[r2], sb);
      const float dw = beta_in[r] * (val[r] - sb);
      out[r] = sm.n_t[r] > 0 ? dw / (float)sm.n_t[r] : 0.f;
    }
  }
}

// dd[m] = <G[m + shift[r(m)]], Z[m]> (warp per merged row)
template <int D>
__global__ void __launch_bounds__(256)
k_sem_dd(SemMeta sm, const float* __restrict__ G, const float* __restrict__ Z,
         float* __restrict__ dd) {
  HF_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int m = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (m >= sm.rows) return;
  int lo = 0, hi = sm.R;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (sm.rel_row_off[mid] <= m) lo = mid; else hi = mid;
  }
  const float* g = G + (long long)(m + sm.shift[lo]) * D;
  const float* z = Z + (long long)m * D;
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < D / 32; k++) acc = fmaf(__ldg(g + lane + 32 * k), __ldg(z + lane + 32 * k), acc);
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) dd[m] = acc;
}

// dWs = Z^T Ga, dbs = column sums of Ga, dq = column sums of Th: chunk c of
// rows -> partial[c] (thread tile (D/16) x (A/16) of dWs; threads < A the
// column sums); then k_sem_wred sums the chunks in order.
constexpr int kSemStage = 32;
template <int D, int A>
__global__ void __launch_bounds__(256)
k_sem_wpart(int rows, int chunk, const float* __restrict__ Z, const float* __restrict__ Ga,
            const float* __restrict__ Th, float* __restrict__ partial) {
  HF_PDL_ENTRY();
  constexpr int DT = D / 16, CT = A / 16;
  __shared__ float zs[kSemStage][D];
  __shared__ float gs[kSemStage][A];
  __shared__ float ts[kSemStage][A];
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  float acc[DT][CT];
#pragma unroll
  for (int i = 0; i < DT; i++)
#pragma unroll
    for (int j = 0; j < CT; j++) acc[i][j] = 0.f;
  float cb = 0.f, cq = 0.f;
  const int r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  for (int b = r0; b < r1; b += kSemStage) {
    const int n = min(kSemStage, r1 - b);
    __syncthreads();
    for (int i = threadIdx.x; i < kSemStage * D; i += 256) {
      const int r = i / D, c = i % D;
      zs[r][c] = r < n ? __ldg(Z + (long long)(b + r) * D + c) : 0.f;
    }
    for (int i = threadIdx.x; i < kSemStage * A; i += 256) {
      const int r = i / A, c = i % A;
      gs[r][c] = r < n ? __ldg(Ga + (long long)(b + r) * A + c) : 0.f;
      ts[r][c] = r < n ? __ldg(Th + (long long)(b + r) * A + c) : 0.f;
    }
    __syncthreads();
    for (int r = 0; r < n; r++) {
      float zv[DT], gv[CT];
#pragma unroll
      for (int i = 0; i < DT; i++) zv[i] = zs[r][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < CT; j++) gv[j] = gs[r][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < DT; i++)
#pragma unroll
        for (int j = 0; j < CT; j++) acc[i][j] = fmaf(zv[i], gv[j], acc[i][j]);
      if (threadIdx.x < A) {
        cb += gs[r][threadIdx.x];
        cq += ts[r][threadIdx.x];
      }
    }
  }
  float* out = partial + (long long)blockIdx.x * (D * A + 2 * A);
#pragma unroll
  for (int i = 0; i < DT; i++)
#pragma unroll
    for (int j = 0; j < CT; j++) out[(ty + 16 * i) * A + tx + 16 * j] = acc[i][j];
  if (threadIdx.x < A) {
    out[D * A + threadIdx.x] = cb;
    out[D * A + A + threadIdx.x] = cq;
  }
}

__global__ void __launch_bounds__(256)
k_sem_wred(int nch, int n, const float* __restrict__ partial, float* __restrict__ dWs, int DA,
           int A, float* __restrict__ dbs, float* __restrict__ dq) {
  HF_PDL_ENTRY();
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int c = 0; c < nch; c++) s += partial[(long long)c * n + i];
  if (i < DA) dWs[i] = s;
  else if (i < DA + A) dbs[i - DA] = s;
  else dq[i - DA - A] = s;
}

static int sem_chunks(int rows) { return std::max(1, std::min(2 * sm_count(), (rows + 63) / 64)); }

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
              (const float4*)d_bias, (float4*)d_H, (const float*)nullptr);
  else if (act == HIFUSE_ACT_NONE)
    HF_LAUNCH(k_fuse<false>, grid, 256, 0, s, f, (const float4*)d_Z, (const float4*)d_R0,
              (const float4*)d_bias, (float4*)d_H, (const float*)nullptr);
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


hifuse_status hifuse_semantic_fuse_bwd_bias(const hifuse_layer_shape* shape, int D,
                                            const float* d_G, float* d_dbias, void* d_ws,
                                            size_t ws_bytes, hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (D != 64 && D != 128) return HIFUSE_ERR_UNSUPPORTED;
  if (!d_dbias || (m.dst_rows > 0 && !d_G)) return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_G) || !aligned16(d_dbias)) return HIFUSE_ERR_ALIGNMENT;
  if (ws_bytes < hifuse_fuse_bwd_ws_bytes(shape, D) || !d_ws) return HIFUSE_ERR_WORKSPACE;
  FuseBwdMeta f;
  make_fbm(m, D, &f);
  cudaStream_t s = st(stream);
  float4* partial = (float4*)d_ws;
  // the same chunks and orders as hifuse_semantic_fuse_bwd's bias: bit-identical
  HF_LAUNCH((k_fuse_bwd_chunks<false, false>), f.chunk_off[m.T], 256, 0, s, f,
            (const float4*)d_G, (const float4*)nullptr, (float4*)nullptr, partial);
  HF_LAUNCH(k_fuse_bwd_bias, m.T, 256, 0, s, f, partial, (float4*)d_dbias);
  return last_cuda();
}

size_t hifuse_sem_att_ws_bytes(const hifuse_layer_shape* shape, int D, int A) {
  LayerMeta m;
  if (make_meta(shape, &m) != HIFUSE_OK) return 0;
  const int nch = sem_chunks(m.rows);
  return carve_bytes(m.rows, 4) * 2 + carve_bytes(HF_MAX_R, 4) +
         carve_bytes((long long)m.rows * A, 4) * 2 +
         carve_bytes((long long)nch * (D * A + 2 * A), 4) + hifuse_fuse_bwd_ws_bytes(shape, D);
}

static bool sem_dims_ok(int D, int A) { return (D == 64 || D == 128) && A == D; }

hifuse_status hifuse_semantic_fuse_att(const hifuse_layer_shape* shape, int D, int A,
                                       hifuse_act act, const float* d_Z, const float* d_R0,
                                       const float* d_bias, const float* d_Ws,
                                       const float* d_bs, const float* d_q, float* d_beta,
                                       float* d_w, float* d_H, void* d_ws, size_t ws_bytes,
                                       hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (!sem_dims_ok(D, A)) return HIFUSE_ERR_UNSUPPORTED;
  if (!d_Ws || !d_bs || !d_q || !d_beta || (m.dst_rows > 0 && !d_H) || (m.rows > 0 && !d_Z))
    return HIFUSE_ERR_INVALID_ARG;
  if (act != HIFUSE_ACT_RELU && act != HIFUSE_ACT_NONE) return HIFUSE_ERR_INVALID_ARG;
  if (!aligned16(d_Z) || !aligned16(d_R0) || !aligned16(d_bias) || !aligned16(d_H))
    return HIFUSE_ERR_ALIGNMENT;
  if (ws_bytes < hifuse_sem_att_ws_bytes(shape, D, A) || !d_ws) return HIFUSE_ERR_WORKSPACE;
  cudaStream_t s = st(stream);
  SemMeta sm;
  make_sem_meta(m, &sm);
  char* p = (char*)d_ws;
  float* sc = carve<float>(p, m.rows);
  const int grid = std::max(1, std::min(sm_count() * 2, (m.rows + kSemWarps * kSemRPW - 1) /
                                                            (kSemWarps * kSemRPW)));
#define HF_SEMF(DD)                                                                            \
  set_max_smem(reinterpret_cast<const void*>(&k_sem_rows<DD, DD, false>), (int)sem_smem<DD, DD>());             \
  HF_LAUNCH((k_sem_rows<DD, DD, false>), grid, kSemWarps * 32, (sem_smem<DD, DD>()), s, sm, d_Z, \
            d_Ws, d_bs, d_q, sc, (const float*)nullptr, (const float*)nullptr,                \
            (const float*)nullptr, (float*)nullptr, (float*)nullptr, (float*)nullptr)
  if (m.rows > 0) { if (D == 128) { HF_SEMF(128); } else { HF_SEMF(64); } }
#undef HF_SEMF
  HF_LAUNCH(k_sem_rel<false>, 1, 256, 0, s, sm, sc, (const float*)nullptr, d_beta, d_w);
  FuseMeta f;
  make_fuse_meta(m, D, &f);
  long long n = (long long)m.dst_rows * (D / 4);
  if (act == HIFUSE_ACT_RELU)
    HF_LAUNCH(k_fuse<true>, ceil_div(n, 256), 256, 0, s, f, (const float4*)d_Z,
              (const float4*)d_R0, (const float4*)d_bias, (float4*)d_H, (const float*)d_beta);
  else
    HF_LAUNCH(k_fuse<false>, ceil_div(n, 256), 256, 0, s, f, (const float4*)d_Z,
              (const float4*)d_R0, (const float4*)d_bias, (float4*)d_H, (const float*)d_beta);
  return last_cuda();
}

hifuse_status hifuse_semantic_fuse_att_bwd(const hifuse_layer_shape* shape, int D, int A,
                                           hifuse_act act, const float* d_dH, const float* d_H,
                                           const float* d_Z, const float* d_Ws,
                                           const float* d_bs, const float* d_q,
                                           const float* d_beta, float* d_G, float* d_dZ,
                                           float* d_dbias, float* d_dWs, float* d_dbs,
                                           float* d_dq, void* d_ws, size_t ws_bytes,
                                           hifuse_stream_t stream) {
  LayerMeta m;
  hifuse_status rc = make_meta(shape, &m);
  if (rc != HIFUSE_OK) return rc;
  if (!sem_dims_ok(D, A)) return HIFUSE_ERR_UNSUPPORTED;
  if (!d_Ws || !d_bs || !d_q || !d_beta || !d_dWs || !d_dbs || !d_dq ||
      (m.rows > 0 && (!d_Z || !d_dZ)) || (m.dst_rows > 0 && (!d_dH || !d_G)) ||
      (act == HIFUSE_ACT_RELU && m.dst_rows > 0 && !d_H))
    return HIFUSE_ERR_INVALID_ARG;
  if (ws_bytes < hifuse_sem_att_ws_bytes(shape, D, A) || !d_ws) return HIFUSE_ERR_WORKSPACE;
  cudaStream_t s = st(stream);
  SemMeta sm;
  make_sem_meta(m, &sm);
  char* p = (char*)d_ws;
  (void)carve<float>(p, m.rows);                       // forward scores (unused here)
  float* dd = carve<float>(p, m.rows);
  float* coef = carve<float>(p, HF_MAX_R);
  float* Ga = carve<float>(p, (long long)m.rows * A);
  float* Th = carve<float>(p, (long long)m.rows * A);
  const int nch = sem_chunks(m.rows);
  float* partial = carve<float>(p, (long long)nch * (D * A + 2 * A));
  const size_t fb = hifuse_fuse_bwd_ws_bytes(shape, D);
  // G = dH act'(H), dbias (A6a)
  rc = hifuse_semantic_fuse_bwd(shape, D, act, d_dH, d_H, d_G, d_dbias, p, fb, stream);
  if (rc != HIFUSE_OK) return rc;
  const int grid = std::max(1, std::min(sm_count() * 2, (m.rows + kSemWarps * kSemRPW - 1) /
                                                            (kSemWarps * kSemRPW)));
  const int chunk = std::max(1, (m.rows + nch - 1) / nch);
#define HF_SEMB(DD)                                                                            \
  if (m.rows > 0) {                                                                             \
    HF_LAUNCH(k_sem_dd<DD>, ceil_div(m.rows, 8), 256, 0, s, sm, d_G, d_Z, dd);                  \
  }                                                                                             \
  HF_LAUNCH(k_sem_rel<true>, 1, 256, 0, s, sm, dd, d_beta, coef, (float*)nullptr);              \
  if (m.rows > 0) {                                                                             \
    set_max_smem(reinterpret_cast<const void*>(&k_sem_rows<DD, DD, true>), (int)sem_smem<DD, DD>());               \
    HF_LAUNCH((k_sem_rows<DD, DD, true>), grid, kSemWarps * 32, (sem_smem<DD, DD>()), s, sm, d_Z, \
              d_Ws, d_bs, d_q, (float*)nullptr, d_G, d_beta, coef, d_dZ, Ga, Th);              \
  }                                                                                             \
  HF_LAUNCH((k_sem_wpart<DD, DD>), nch, 256, 0, s, m.rows, chunk, d_Z, Ga, Th, partial)
  if (D == 128) { HF_SEMB(128); } else { HF_SEMB(64); }
#undef HF_SEMB
  const int nout = D * A + 2 * A;
  HF_LAUNCH(k_sem_wred, ceil_div(nout, 256), 256, 0, s, nch, nout, partial, d_dWs, D * A, A,
            d_dbs, d_dq);
  return last_cuda();
}

}  // extern "C"

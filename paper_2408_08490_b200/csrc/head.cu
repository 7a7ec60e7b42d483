// head.cu -- training-step helpers outside the paper's four HGNN stages:
// the linear classifier with mean softmax cross-entropy on the seed rows
// (closes the loop of PAPER.md line 156 "forward ... backward
// ... parameter update") and the SGD update.  Deterministic fixed-order sums.
//
// Three kernels for the classifier:
//  k_head_logits  logits = Hs Wc + bc
//  k_head_softmax warp per seed row: dlog = (softmax - onehot) / B, row loss;
//                 the last block sums the per-block losses -> mean loss
//  k_head_grads   one grid, two jobs: dHs = dlog Wc^T and dWc = Hs^T dlog
//                 (+ dbc = column sums of dlog), each output tile split over
//                 K across the 8 CTAs of a thread-block cluster whose
//                 partials are summed in rank order through distributed
//                 shared memory.
// The three GEMMs run on the tensor cores with mma.sync m16n8k8 TF32 in the
// 3xTF32 split (x = hi + lo, hi = tf32(x), lo = tf32(x - hi); D += lo*hi +
// hi*lo + hi*hi), which keeps fp32-level accuracy: the head is outside the
// paper's stages and must not add TF32 error to the fp32 step.  These GEMMs
// are tiny (B x 128 x C); what matters is parallelism and few dependent
// memory round trips, not the tcgen05 peak.
#include <algorithm>
#include <cooperative_groups.h>
#include "common.cuh"

namespace hf {

#ifndef HF_HEAD_BK
#define HF_HEAD_BK 32
#endif
static constexpr int kBK = HF_HEAD_BK;     // K slab
static constexpr int kBM = 32, kBN = 64;   // block tile; 4 warps of 16 x 32

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma_tf32_16x8x8(float (&d)[4], const uint32_t (&a)[4],
                                                const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// One kBM x kBN tile of C = op(A) op(B) over k in [kb0, kb1) on 128 threads:
// TA: A stored [K][M] (else [M][K]); TB: B stored [N][K] (else [K][N]).  Warp w
// owns rows 16 (w / 2) .. +16 and columns 32 (w % 2) .. +32 (4 n-tiles of 8);
// acc[nt][4] in the mma C-fragment layout.  K slabs are staged in shared
// memory (padded: conflict-free fragment reads), the next slab prefetched
// into registers.  colsum != nullptr: threads 0..kBN-1 also return
// sum_k B[k][n0 + tid] there.
template <bool TA, bool TB>
__device__ __forceinline__ void mma_tile(int M, int N, const float* __restrict__ A, int lda,
                                         const float* __restrict__ B, int ldb, int m0, int n0,
                                         int kb0, int kb1, float (&acc)[4][4], float* colsum) {
  __shared__ float As[kBM][kBK + 4];
  __shared__ float Bs[kBK][kBN + 8];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (w >> 1) * 16, wn = (w & 1) * 32;
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0.f;
  float cs = 0.f;
  constexpr int QA = kBM * kBK / 128, QB = kBK * kBN / 128;   // slab loads per thread
  float ra[QA], rb[QB];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int q = 0; q < QA; q++) {                // A slab: kBM x kBK
      const int i = tid + 128 * q;
      const int kk = TA ? i / kBM : i % kBK, mm = TA ? i % kBM : i / kBK;
      const int m = m0 + mm, k = k0 + kk;
      ra[q] = (m < M && k < kb1) ? (TA ? A[(long long)k * lda + m] : A[(long long)m * lda + k]) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < QB; q++) {                // B slab: kBK x kBN
      const int i = tid + 128 * q;
      const int kk = TB ? i % kBK : i / kBN, nn = TB ? i / kBK : i % kBN;
      const int n = n0 + nn, k = k0 + kk;
      rb[q] = (n < N && k < kb1) ? (TB ? B[(long long)n * ldb + k] : B[(long long)k * ldb + n]) : 0.f;
    }
  };
  if (kb0 < kb1) fetch(kb0);
  for (int k0 = kb0; k0 < kb1; k0 += kBK) {
#pragma unroll
    for (int q = 0; q < QA; q++) {
      const int i = tid + 128 * q;
      As[TA ? i % kBM : i / kBK][TA ? i / kBM : i % kBK] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < QB; q++) {
      const int i = tid + 128 * q;
      Bs[TB ? i % kBK : i / kBN][TB ? i / kBK : i % kBN] = rb[q];
    }
    __syncthreads();
    if (k0 + kBK < kb1) fetch(k0 + kBK);
    if (colsum && tid < kBN) {
#pragma unroll 8
      for (int kk = 0; kk < kBK; kk++) cs += Bs[kk][tid];
    }
#pragma unroll
    for (int ks = 0; ks < kBK; ks += 8) {
      uint32_t ah[4], al[4];
      const float av[4] = {As[wm + g][ks + t], As[wm + g + 8][ks + t], As[wm + g][ks + t + 4],
                           As[wm + g + 8][ks + t + 4]};
#pragma unroll
      for (int r = 0; r < 4; r++) {
        ah[r] = to_tf32(av[r]);
        al[r] = to_tf32(av[r] - __uint_as_float(ah[r]));
      }
#pragma unroll
      for (int nt = 0; nt < 4; nt++) {
        const int n = wn + nt * 8 + g;
        const float bv[2] = {Bs[ks + t][n], Bs[ks + t + 4][n]};
        uint32_t bh[2], bl[2];
#pragma unroll
        for (int r = 0; r < 2; r++) {
          bh[r] = to_tf32(bv[r]);
          bl[r] = to_tf32(bv[r] - __uint_as_float(bh[r]));
        }
        mma_tf32_16x8x8(acc[nt], al, bh);
        mma_tf32_16x8x8(acc[nt], ah, bl);
        mma_tf32_16x8x8(acc[nt], ah, bh);
      }
    }
    __syncthreads();
  }
  if (colsum && tid < kBN) *colsum = cs;
}

// C-fragment coordinates of acc[nt][r], relative to the tile
__device__ __forceinline__ int frag_row(int r) {
  return ((threadIdx.x >> 5) >> 1) * 16 + ((threadIdx.x & 31) >> 2) + (r >= 2 ? 8 : 0);
}
__device__ __forceinline__ int frag_col(int nt, int r) {
  return ((threadIdx.x >> 5) & 1) * 32 + nt * 8 + (threadIdx.x & 3) * 2 + (r & 1);
}

__global__ void __launch_bounds__(128)
k_head_logits(int B, int D, int C, const float* __restrict__ Hs, const float* __restrict__ Wc,
              const float* __restrict__ bc, float* __restrict__ lg, int* __restrict__ tickets,
              int ntickets) {
  HF_PDL_ENTRY();
  if (blockIdx.x == 0 && blockIdx.y == 0)   // tickets of the next two kernels
    for (int i = threadIdx.x; i < ntickets; i += blockDim.x) tickets[i] = 0;
  float acc[4][4];
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
  mma_tile<false, false>(B, C, Hs, D, Wc, C, m0, n0, 0, D, acc, nullptr);
#pragma unroll
  for (int nt = 0; nt < 4; nt++)
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int m = m0 + frag_row(r), n = n0 + frag_col(nt, r);
      if (m < B && n < C) lg[(long long)m * C + n] = acc[nt][r] + __ldg(bc + n);
    }
}

// 8 rows (one per warp) per block; lg is turned into dlog in place.  NV > 0:
// the row (C <= 32 NV) is loaded once into registers with all loads in flight
// together (the loops of the generic NV = 0 path are latency-bound: one
// dependent L2 round trip per 32 columns per pass).
template <int NV>
__global__ void __launch_bounds__(256)
k_head_softmax(int B, int C, const int* __restrict__ labels, float* __restrict__ lg,
               float* __restrict__ block_loss, int* __restrict__ ticket, float* __restrict__ loss,
               int* __restrict__ status) {
  HF_PDL_ENTRY();
  __shared__ float s_l[8];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = blockIdx.x * 8 + w;
  float rl = 0.f;
  if (b < B) {
    float* x = lg + (long long)b * C;
    // a label outside [0, C) drops the row (no loss term, zero gradient) and
    // sets HIFUSE_ST_BAD_LABEL; it is never used as an index
    const int y0 = labels[b];
    const bool ok = (unsigned)y0 < (unsigned)C;
    const int y = ok ? y0 : 0;
    if (!ok && lane == 0 && status) atomicOr(status, HIFUSE_ST_BAD_LABEL);
    const float inv = ok ? 1.f / (float)B : 0.f;
    float mx = -INFINITY, se = 0.f, ly;
    if constexpr (NV > 0) {
      float v[NV];
#pragma unroll
      for (int q = 0; q < NV; q++) {
        const int c = lane + 32 * q;
        v[q] = c < C ? x[c] : -INFINITY;
      }
      {
        // the label's raw logit: owner lane y % 32, register y / 32
        float e = 0.f;
#pragma unroll
        for (int q = 0; q < NV; q++)
          if (q == (y >> 5)) e = v[q];
        ly = __shfl_sync(0xffffffffu, e, y & 31);
      }
#pragma unroll
      for (int q = 0; q < NV; q++) mx = fmaxf(mx, v[q]);
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
#pragma unroll
      for (int q = 0; q < NV; q++) {
        v[q] = expf(v[q] - mx);          // exp(-inf) = 0 for the padding
        se += v[q];
      }
      for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
#pragma unroll
      for (int q = 0; q < NV; q++) {
        const int c = lane + 32 * q;
        if (c < C) x[c] = (v[q] / se - (c == y ? 1.f : 0.f)) * inv;
      }
      rl = ok ? logf(se) + mx - ly : 0.f;
    } else {
      for (int c = lane; c < C; c += 32) mx = fmaxf(mx, x[c]);
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      for (int c = lane; c < C; c += 32) se += expf(x[c] - mx);
      for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      ly = x[y];
      __syncwarp();
      for (int c = lane; c < C; c += 32) x[c] = (expf(x[c] - mx) / se - (c == y ? 1.f : 0.f)) * inv;
      rl = ok ? logf(se) + mx - ly : 0.f;
    }
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

// Few classes (C <= 32, the RGCN/RGAT configs except ogbn-mag): the whole
// critical part of the head in ONE kernel, one warp per seed row:
//   lane c < C: logit_c = bc_c + <Hs_b, Wc[:, c]> (Hs row broadcast by shuffles,
//   Wc is a few KB and stays in L1) -> softmax / cross-entropy across the lanes
//   -> dlog (global, for hifuse_linear_xent_wgrad) -> dHs_b[k] = sum_c dlog_c
//   Wc[k, c] (lane k + 32 j).  Exact fp32; replaces three latency-bound
//   launches.  Block = 8 rows; the last block sums the per-block losses.
template <int D, int CMAX>
__global__ void __launch_bounds__(256)
k_head_small(int B, int C, const float* __restrict__ Hs, const float* __restrict__ Wc,
             const float* __restrict__ bc, const int* __restrict__ labels,
             float* __restrict__ dlog, float* __restrict__ dHs, float* __restrict__ block_loss,
             int* __restrict__ ticket, float* __restrict__ loss, int* __restrict__ status) {
  HF_PDL_ENTRY();
  constexpr int KPL = D / 32;              // features per lane
  __shared__ float s_l[8];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = blockIdx.x * 8 + w;
  float rl = 0.f;
  if (b < B) {
    float hv[KPL];
#pragma unroll
    for (int j = 0; j < KPL; j++) hv[j] = Hs[(long long)b * D + j * 32 + lane];
    const bool act = lane < C;
    // lane owns features k = lane + 32 j: partial logits of every class over
    // its features, then one butterfly sum per class (no serial K chain)
    float pc[CMAX];
#pragma unroll
    for (int c = 0; c < CMAX; c++) pc[c] = 0.f;
#pragma unroll
    for (int j = 0; j < KPL; j++) {
      const float* wr = Wc + (long long)(j * 32 + lane) * C;
#pragma unroll
      for (int c = 0; c < CMAX; c++)
        if (c < C) pc[c] = fmaf(hv[j], __ldg(wr + c), pc[c]);
    }
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < CMAX; c++) {
      if (c >= C) break;
      float v = pc[c];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == c) acc = v;
    }
    float z = act ? __ldg(bc + lane) : -INFINITY;
    if (act) z += acc;
    float mx = z;
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float ex = act ? expf(z - mx) : 0.f;
    float se = ex;
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    // a label outside [0, C) drops the row (HIFUSE_ST_BAD_LABEL)
    const int y0 = labels[b];
    const bool ok = (unsigned)y0 < (unsigned)C;
    const int y = ok ? y0 : 0;
    if (!ok && lane == 0 && status) atomicOr(status, HIFUSE_ST_BAD_LABEL);
    const float zy = __shfl_sync(0xffffffffu, z, y);
    const float g = act && ok ? (ex / se - (lane == y ? 1.f : 0.f)) / (float)B : 0.f;
    if (act) dlog[(long long)b * C + lane] = g;
    rl = ok ? logf(se) + mx - zy : 0.f;
#pragma unroll
    for (int j = 0; j < KPL; j++) {
      const int k = j * 32 + lane;
      float d = 0.f;
      for (int c = 0; c < C; c++)
        d = fmaf(__shfl_sync(0xffffffffu, g, c), __ldg(Wc + (long long)k * C + c), d);
      dHs[(long long)b * D + k] = d;
    }
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

__global__ void k_zero_int(int* p) {
  HF_PDL_ENTRY(); *p = 0; }

struct HeadGrid {
  int dh_tiles_n, dh_tiles;       // dHs: [B, D] tiles (n-major), K = C
  int dw_tiles_n, dw_tiles;       // dWc: [D, C] tiles, K = B
};

// One thread-block cluster of kSlices CTAs per output tile: CTA rank z
// computes the partial product over its K slice, the partials meet in
// distributed shared memory and each rank sums 1/kSlices of the tile over the
// ranks in rank order (deterministic; no global partials, no atomics).
static constexpr int kSlices = 8;

__global__ void __cluster_dims__(kSlices, 1, 1) __launch_bounds__(128)
k_head_grads(int B, int D, int C, HeadGrid hg, const float* __restrict__ Hs,
             const float* __restrict__ Wc, const float* __restrict__ dlog,
             float* __restrict__ dHs, float* __restrict__ dWc, float* __restrict__ dbc) {
  HF_PDL_ENTRY();
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ float red[128 * 16];      // this CTA's partial, [thread][16 fragment values]
  __shared__ float red_b[kBN];         // this CTA's column sums (dbc tiles)
  const int z = (int)cluster.block_rank();
  const int tile = blockIdx.x / kSlices;
  const bool dh = tile < hg.dh_tiles;
  int M, N, ld, m0, n0;
  float* out;
  float acc[4][4];
  bool bias = false;
  if (dh) {
    // ---- dHs = dlog Wc^T: M = B, N = D, K = C; Wc stored [D][C] = [N][K]
    M = B; N = D; ld = D; out = dHs;
    m0 = (tile / hg.dh_tiles_n) * kBM;
    n0 = (tile % hg.dh_tiles_n) * kBN;
    const int kper = ((C + kSlices - 1) / kSlices + kBK - 1) / kBK * kBK;
    mma_tile<false, true>(B, D, dlog, C, Wc, C, m0, n0, z * kper, min(C, (z + 1) * kper), acc,
                          nullptr);
  } else {
    // ---- dWc = Hs^T dlog: M = D, N = C, K = B; Hs stored [B][D] = [K][M]
    const int t2 = tile - hg.dh_tiles;
    M = D; N = C; ld = C; out = dWc;
    m0 = (t2 / hg.dw_tiles_n) * kBM;
    n0 = (t2 % hg.dw_tiles_n) * kBN;
    const int kper = ((B + kSlices - 1) / kSlices + kBK - 1) / kBK * kBK;
    bias = m0 == 0;                    // the first row tile also forms dbc
    float cs = 0.f;
    mma_tile<true, false>(D, C, Hs, D, dlog, C, m0, n0, z * kper, min(B, (z + 1) * kper), acc,
                          bias ? &cs : nullptr);
    if (bias && threadIdx.x < kBN) red_b[threadIdx.x] = cs;
  }
#pragma unroll
  for (int nt = 0; nt < 4; nt++)
#pragma unroll
    for (int r = 0; r < 4; r++) red[threadIdx.x * 16 + nt * 4 + r] = acc[nt][r];
  cluster.sync();
  // rank z reduces the fragments of threads [16 z, 16 z + 16): 256 values,
  // two per thread, each summed over the kSlices ranks in rank order
  {
    const int ot = z * 16 + (threadIdx.x >> 3);        // owning thread of the fragment
    const int q0 = (threadIdx.x & 7) * 2;              // its values q0, q0 + 1
    float v[2][kSlices];
#pragma unroll
    for (int rk = 0; rk < kSlices; rk++) {
      const float* peer = cluster.map_shared_rank(red, rk);
      v[0][rk] = peer[ot * 16 + q0];
      v[1][rk] = peer[ot * 16 + q0 + 1];
    }
#pragma unroll
    for (int u = 0; u < 2; u++) {
      float t = 0.f;
#pragma unroll
      for (int rk = 0; rk < kSlices; rk++) t += v[u][rk];
      const int q = q0 + u, nt = q >> 2, r = q & 3;
      // fragment coordinates of thread ot
      const int w = ot >> 5, ln = ot & 31;
      const int m = m0 + (w >> 1) * 16 + (ln >> 2) + (r >= 2 ? 8 : 0);
      const int n = n0 + (w & 1) * 32 + nt * 8 + (ln & 3) * 2 + (r & 1);
      if (m < M && n < N) out[(long long)m * ld + n] = t;
    }
  }
  if (bias && z == 0 && threadIdx.x < kBN && n0 + (int)threadIdx.x < C) {
    float t = 0.f;
#pragma unroll
    for (int rk = 0; rk < kSlices; rk++) t += cluster.map_shared_rank(red_b, rk)[threadIdx.x];
    dbc[n0 + threadIdx.x] = t;
  }
  cluster.sync();                      // peers' shared memory stays alive until read
}

static HeadGrid head_grid(int B, int D, int C) {
  (void)B;
  HeadGrid h;
  h.dh_tiles_n = (int)ceil_div(D, kBN);
  h.dh_tiles = h.dh_tiles_n * (int)ceil_div(B, kBM);
  h.dw_tiles_n = (int)ceil_div(C, kBN);
  h.dw_tiles = h.dw_tiles_n * (int)ceil_div(D, kBM);
  return h;
}

__global__ void k_sgd(float4* __restrict__ p, const float4* __restrict__ g, long long n4, float lr) {
  HF_PDL_ENTRY();
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  float4 a = p[i], b = g[i];
  a.x -= lr * b.x; a.y -= lr * b.y; a.z -= lr * b.z; a.w -= lr * b.w;
  p[i] = a;
}

__global__ void k_sgd_tail(float* __restrict__ p, const float* __restrict__ g, long long from,
                           long long n, float lr) {
  HF_PDL_ENTRY();
  long long i = from + threadIdx.x;
  if (i < n) p[i] -= lr * g[i];
}

}  // namespace hf

using namespace hf;

extern "C" {

size_t hifuse_xent_ws_bytes(int B, int D, int C) {
  if (B <= 0 || D <= 0 || C <= 0) return 0;
  return carve_bytes((long long)B * C, 4) + carve_bytes(ceil_div(B, 8), 4) + carve_bytes(1, 4);
}

hifuse_status hifuse_linear_xent(int B, int D, int C, const float* d_H, int64_t h_rows,
                                 int64_t h_row0, const int32_t* d_labels, const float* d_Wc,
                                 const float* d_bc, float* d_loss, float* d_dH, float* d_dWc,
                                 float* d_dbc, void* d_ws, size_t ws_bytes, int32_t* d_status,
                                 hifuse_stream_t stream) {
  if (B <= 0 || D <= 0 || C <= 0 || h_row0 < 0 || h_row0 + B > h_rows || !d_H || !d_labels ||
      !d_Wc || !d_bc || !d_loss || !d_dH || (!d_dWc != !d_dbc))
    return HIFUSE_ERR_INVALID_ARG;
  if (ws_bytes < hifuse_xent_ws_bytes(B, D, C) || !d_ws) return HIFUSE_ERR_WORKSPACE;
  cudaStream_t s = st(stream);
  HeadGrid h = head_grid(B, D, C);
  const int nblk = (int)ceil_div(B, 8);
  char* p = (char*)d_ws;
  float* dlog = carve<float>(p, (long long)B * C);
  float* block_loss = carve<float>(p, nblk);
  int* ticket = carve<int>(p, 1);
  // rows of dH outside the seeds get no gradient
  if (h_row0 > 0) cudaMemsetAsync(d_dH, 0, sizeof(float) * h_row0 * D, s);
  if (h_row0 + B < h_rows)
    cudaMemsetAsync(d_dH + (h_row0 + B) * D, 0, sizeof(float) * (h_rows - h_row0 - B) * D, s);
  const float* Hs = d_H + h_row0 * D;
  if (C <= 32 && (D == 128 || D == 64)) {
    HF_LAUNCH(k_zero_int, 1, 1, 0, s, ticket);
#define HF_SMALL(DD, CC)                                                                      \
  HF_LAUNCH((k_head_small<DD, CC>), nblk, 256, 0, s, B, C, Hs, d_Wc, d_bc, d_labels, dlog,      \
            d_dH + h_row0 * D, block_loss, ticket, d_loss, d_status)
    if (D == 128) { if (C <= 8) HF_SMALL(128, 8); else HF_SMALL(128, 32); }
    else { if (C <= 8) HF_SMALL(64, 8); else HF_SMALL(64, 32); }
#undef HF_SMALL
    h.dh_tiles = 0;                    // dHs done
    if (!d_dWc) h.dw_tiles = 0;
    if (h.dw_tiles)
      HF_LAUNCH(k_head_grads, h.dw_tiles * kSlices, 128, 0, s, B, D, C, h, Hs, d_Wc, dlog,
                d_dH + h_row0 * D, d_dWc, d_dbc);
    return last_cuda();
  }
  HF_LAUNCH(k_head_logits, dim3(ceil_div(C, kBN), ceil_div(B, kBM)), 128, 0, s, B, D, C, Hs,
            d_Wc, d_bc, dlog, ticket, 1);
  if (C <= 128)
    HF_LAUNCH(k_head_softmax<4>, nblk, 256, 0, s, B, C, d_labels, dlog, block_loss, ticket,
              d_loss, d_status);
  else if (C <= 512)
    HF_LAUNCH(k_head_softmax<16>, nblk, 256, 0, s, B, C, d_labels, dlog, block_loss, ticket,
              d_loss, d_status);
  else
    HF_LAUNCH(k_head_softmax<0>, nblk, 256, 0, s, B, C, d_labels, dlog, block_loss, ticket,
              d_loss, d_status);
  if (!d_dWc) h.dw_tiles = 0;          // weight gradient deferred to hifuse_linear_xent_wgrad
  HF_LAUNCH(k_head_grads, (h.dh_tiles + h.dw_tiles) * kSlices, 128, 0, s, B, D, C, h, Hs, d_Wc,
            dlog, d_dH + h_row0 * D, d_dWc, d_dbc);
  return last_cuda();
}

hifuse_status hifuse_linear_xent_wgrad(int B, int D, int C, const float* d_H, int64_t h_rows,
                                       int64_t h_row0, float* d_dWc, float* d_dbc, void* d_ws,
                                       size_t ws_bytes, hifuse_stream_t stream) {
  if (B <= 0 || D <= 0 || C <= 0 || h_row0 < 0 || h_row0 + B > h_rows || !d_H || !d_dWc ||
      !d_dbc)
    return HIFUSE_ERR_INVALID_ARG;
  if (ws_bytes < hifuse_xent_ws_bytes(B, D, C) || !d_ws) return HIFUSE_ERR_WORKSPACE;
  HeadGrid h = head_grid(B, D, C);
  h.dh_tiles = 0;
  char* p = (char*)d_ws;
  const float* dlog = carve<float>(p, (long long)B * C);
  HF_LAUNCH(k_head_grads, h.dw_tiles * kSlices, 128, 0, st(stream), B, D, C, h, d_H + h_row0 * D,
            (const float*)nullptr, dlog, (float*)nullptr, d_dWc, d_dbc);
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

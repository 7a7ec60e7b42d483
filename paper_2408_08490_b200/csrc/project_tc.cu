// project_tc.cu -- A3 projection on the 5th-generation tensor cores:
// tcgen05.mma kind::tf32, fp32 accumulators in TMEM (readings C17/C18).
//
// Grouped GEMM: every 128-row output tile belongs to one group (relation r:
// compact Y rows, A rows gathered through y_src [and gather_ids for layer 0,
// i.e. the feature collection A2 is fused into the operand load]; or root
// type t: the destination prefix of X_t).  Per tile:
//   * 128 threads; thread t owns output row t of the tile;
//   * K is streamed in 32-element (128-byte) chunks through a 2-stage shared
//     memory ring; A rows are gathered with 16-byte cp.async straight into the
//     128B-swizzled K-major layout the MMA descriptors describe; B = W_g^T
//     (pre-transposed to [D][K], K-major) the same way;
//   * one elected thread issues 4 tcgen05.mma (M=128, N=D, K=8) per chunk and
//     commits them to the stage's mbarrier, which frees the stage;
//   * epilogue: warp w reads TMEM lanes 32w..32w+31 (its 32 rows) with
//     tcgen05.ld and stores fp32 rows.
// The projection is HBM-bound at K = D = 64/128 (32 flop/B), so the design
// goal is streaming A at full bandwidth with enough CTAs per SM (64 KB smem,
// <=128 TMEM columns each -> 3-4 CTAs/SM) rather than peak MMA rate.
#include <algorithm>
#include <cuda_bf16.h>
#include <cstdlib>
#include "project.cuh"
#include "tc_common.cuh"

namespace hf {

using namespace tc;

// 8 fp32 -> 8 bf16 (RN-even, cvt.rn.bf16x2) -> one 16-byte shared store
__device__ __forceinline__ void st_shared_bf16x8(uint32_t dst, float4 a, float4 b) {
  uint32_t w[4];
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w[0]) : "f"(a.y), "f"(a.x));
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w[1]) : "f"(a.w), "f"(a.z));
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w[2]) : "f"(b.y), "f"(b.x));
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w[3]) : "f"(b.w), "f"(b.z));
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(w[0]), "r"(w[1]),
               "r"(w[2]), "r"(w[3])
               : "memory");
}

__device__ __forceinline__ bool tc_resolve(const ProjMeta& pm, const int* table,
                                           const int* rel_y_off, int bid, int step, int* g_out,
                                           int* r0, int* nrows) {
  int G = pm.R + pm.T;
  if (bid >= table[G]) return false;
  int lo = 0, hi = G;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (table[mid] <= bid) lo = mid; else hi = mid;
  }
  int g = lo;
  int total = g < pm.R ? rel_y_off[g + 1] - rel_y_off[g] : pm.n_dst[g - pm.R];
  int local0 = (bid - table[g]) * step;
  *g_out = g;
  *r0 = local0;
  *nrows = min(step, total - local0);
  return *nrows > 0;
}

// A row of group g, local row j.  direct (aggregate-first input): message
// group rows are the aggregated rows rel_off[g] + j of Xm, never gathered.
__device__ __forceinline__ long long tc_a_row(const ProjMeta& pm, const int* rel_y_off,
                                              const int* y_src, const int* gather_ids, int g,
                                              int j, bool direct = false) {
  int x;
  if (g < pm.R && direct) return (long long)rel_y_off[g] + j;
  if (g < pm.R) x = pm.type_src_off[pm.rel_src[g]] + y_src[rel_y_off[g] + j];
  else x = pm.type_src_off[g - pm.R] + j;
  return gather_ids ? (long long)gather_ids[x] : (long long)x;
}

}  // namespace hf

namespace hf {

// ----------------------------------------------------------------- dgrad ----
// Tile = 128 source rows of one type s x KN output features (the K output
// columns split into NS = K / KN CTAs, so a small layer still puts two CTAs
// and twice the loads in flight on every SM); the "K loop" runs over the
// terms (relations out of s, then the root weight) x D/32 chunks.  A chunk:
// 32 columns of dYt rows gathered through slot_y (zero rows where the source
// has no edge of that relation); B chunk: W_term[k][d0..d0+32) for the CTA's
// KN features k, which is already K-major (row k contiguous in d).
#ifndef HF_DG_STAGES
#define HF_DG_STAGES 6
#endif
#ifndef HF_DG_PRODUCERS
#define HF_DG_PRODUCERS 6
#endif
static constexpr int kDgStages = HF_DG_STAGES;
// producer warps: each keeps one chunk in flight (it waits for its own
// cp.async group before arriving), so the chunks in flight per CTA = the
// producer count (4 -> 6 with 6 stages: the mag inner-layer dgrad is one
// 128-row tile per CTA, bound by this load latency)
static constexpr int kDgProd = HF_DG_PRODUCERS;
static_assert(kDgProd >= 4 && kDgProd <= kDgStages, "producers: >= 4 (epilogue), <= stages");

template <int K, int D, int KN, int ST, int PR>
__global__ void __launch_bounds__((PR + 1) * 32)
k_dgrad_tc(DgradMeta dm, const int* __restrict__ slot_y, const float* __restrict__ dY,
           const float* __restrict__ G, const float* __restrict__ W_rel,
           const float* __restrict__ W_root, float* __restrict__ dX, int max_out) {
  HF_PDL_ENTRY();
  // warps 0-3: producers, whole chunks round-robin (warp w loads chunks
  //            w, w + 4, ...: up to four chunks in flight even though each
  //            warp waits for its own cp.async group before the proxy fence);
  //            afterwards the epilogue (TMEM lanes 32w .. 32w + 31)
  // warp 4:    one thread issues the MMAs in chunk order
  constexpr int BM = 128, DC = D / 32, NS = K / KN, P = PR;
  constexpr uint32_t A_STAGE = BM * 128, B_STAGE = KN * 128, STAGE = A_STAGE + B_STAGE;
  constexpr uint32_t IDESC = idesc_tf32(BM, KN, 0, 0);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[ST], empty[ST], done;
  __shared__ uint32_t tmem_slot;
  const int tile = blockIdx.x / NS, n0 = (blockIdx.x % NS) * KN;
  const int s_ = upper_bound_i(dm.tile_off, dm.T + 1, tile) - 1;
  const int j0 = (tile - dm.tile_off[s_]) * BM;
  const int nrows = min(BM, dm.n_src[s_] - j0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  int* s_arow = reinterpret_cast<int*>(smem_raw + (base - smem_u32(smem_raw)) + ST * STAGE);
  if (tid == 0) {
    for (int q = 0; q < ST; q++) {
      mbar_init(smem_u32(&full[q]), 32);
      mbar_init(smem_u32(&empty[q]), 1);
    }
    mbar_init(smem_u32(&done), 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_slot), KN < 32 ? 32 : KN);
  const int nout = dm.out_off[s_ + 1] - dm.out_off[s_];
  const int nterm = nout + (dm.has_root ? 1 : 0);
  const int NC = nterm * DC;
  // dYt row of every (term, tile row), fetched once up front with all loads in
  // flight
  if (tid < BM) {
    const int j = j0 + tid;
    for (int t0 = 0; t0 < nout; t0 += 8) {
      int v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int term = t0 + u;
        v[u] = (term < nout && tid < nrows)
                   ? slot_y[dm.slot_off[dm.out_rel[dm.out_off[s_] + term]] + j] : -1;
      }
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (t0 + u < nout) s_arow[(t0 + u) * BM + tid] = v[u];
    }
  }
  (void)max_out;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp < P) {
    // ------------------------------------------------------------ producers
    for (int c = warp; c < NC; c += P) {
      const int st = c % ST;
      if (c >= ST) mbar_wait(smem_u32(&empty[st]), ((c / ST) - 1) & 1);
      const int term = c / DC, d0 = (c % DC) * 32;
      const bool root = term == nout;
      const float* W;
      if (root) W = W_root + (long long)s_ * K * D;
      else W = W_rel + (long long)dm.out_rel[dm.out_off[s_] + term] * K * D;
      const float* A = root ? G : dY;
      const uint32_t sa = base + st * STAGE, sb = sa + A_STAGE;
#pragma unroll
      for (int i = 0; i < BM / 32; i++) {
        const int r = lane + 32 * i;
        long long a = -1;
        if (root) {
          if (r < nrows && j0 + r < dm.n_dst[s_]) a = (long long)dm.type_dst_off[s_] + j0 + r;
        } else {
          a = s_arow[term * BM + r];
        }
        if (a >= 0) {
          const float* arow = A + a * D + d0;
#pragma unroll
          for (int q = 0; q < 8; q++) cp_async16(sa + sw128_off(r, q), arow + q * 4, 16u);
        } else {        // absent row: zeros by plain shared stores (no zero-fill copies)
#pragma unroll
          for (int q = 0; q < 8; q++)
            asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(sa + sw128_off(r, q)), "r"(0));
        }
      }
#pragma unroll
      for (int i = 0; i < KN / 32; i++) {
        const int r = lane + 32 * i;
        const float* brow = W + (long long)(n0 + r) * D + d0;
#pragma unroll
        for (int q = 0; q < 8; q++) cp_async16(sb + sw128_off(r, q), brow + q * 4, 16);
      }
      cp_async_commit();
      cp_async_wait<0>();
      fence_proxy_async();
      mbar_arrive(smem_u32(&full[st]));
    }
  } else if (lane == 0) {
    // ------------------------------------------------------------------ MMA
    for (int c = 0; c < NC; c++) {
      const int st = c % ST;
      mbar_wait(smem_u32(&full[st]), (c / ST) & 1);
      tc_fence_after();
      const uint32_t sa = base + st * STAGE, sb = sa + A_STAGE;
#pragma unroll
      for (int k = 0; k < 4; k++)
        mma_tf32(tmem, sw128_desc(sa + k * 32, 16, 1024), sw128_desc(sb + k * 32, 16, 1024), IDESC,
                 (c | k) ? 1u : 0u);
      mma_commit(smem_u32(&empty[st]));
    }
    mma_commit(smem_u32(&done));
  }
  __syncwarp();
  if (warp < 4) {
    // -------------------------------------------- epilogue (TMEM lanes 32w..)
    if (NC > 0) {
      mbar_wait(smem_u32(&done), 0);
      tc_fence_after();
    }
    const int row = warp * 32 + lane;
    float* orow = dX + (long long)(dm.type_src_off[s_] + j0 + row) * K + n0;
#pragma unroll
    for (int c0 = 0; c0 < KN; c0 += 16) {
      float v[16];
      if (NC > 0) {
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
      } else {
#pragma unroll
        for (int q = 0; q < 16; q++) v[q] = 0.f;
      }
      if (row < nrows) {
        float4* o = reinterpret_cast<float4*>(orow + c0);
        o[0] = make_float4(v[0], v[1], v[2], v[3]);
        o[1] = make_float4(v[4], v[5], v[6], v[7]);
        o[2] = make_float4(v[8], v[9], v[10], v[11]);
        o[3] = make_float4(v[12], v[13], v[14], v[15]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, KN < 32 ? 32 : KN);
}

__device__ __forceinline__ void group_table_warp(const ProjMeta& pm, const int* s_yoff, int step,
                                                 int* s_tab, int lane);

// ----------------------------------------------------------------- wgrad ----
// Chunk = up to CH rows of one group (CH adapts to the layer size, 128..1024); partial[chunk] = A^T B over the rows,
// A = X rows (features = M, padded to 128 when K = 64), B = dYt / G rows
// (N = D).  The reduction runs over rows, so both operands are MN-major
// (SWIZZLE_128B_BASE32B): a stage holds 32 rows; per 32-feature block the 32
// rows are 8 atoms of 4 rows x 128 B (512 B each, SBO = 512), blocks at
// LBO = 4096; each 16-byte cp.async (4 features of one row) lands inside one
// swizzled 32-byte chunk.
static constexpr int kWgStages = 3;

template <int K, int D>
__global__ void __launch_bounds__(128)
k_wgrad_tc(ProjMeta pm, int CH, const int* __restrict__ chunk_off, const int* __restrict__ rel_y_off,
           const int* __restrict__ y_src, const int* __restrict__ gather_ids,
           const float* __restrict__ X, const float* __restrict__ dY, const float* __restrict__ G,
           float* __restrict__ partial, const float* __restrict__ Xm) {
  HF_PDL_ENTRY();
  constexpr int MA = 128;                               // padded M (features)
  constexpr uint32_t BLK = 4096;                        // one 32-feature block of 32 rows
  constexpr uint32_t A_STAGE = (MA / 32) * BLK, B_STAGE = (D / 32) * BLK, STAGE = A_STAGE + B_STAGE;
  constexpr uint32_t IDESC = idesc_tf32(MA, D, 1, 1);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[kWgStages];
  __shared__ uint32_t tmem_slot;
  __shared__ int s_tab[HF_MAX_R + HF_MAX_T + 1], s_yo[HF_MAX_R + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i <= pm.R; i += blockDim.x) s_yo[i] = rel_y_off[i];
  __syncthreads();
  if (warp == 0) group_table_warp(pm, s_yo, CH, s_tab, lane);
  __syncthreads();
  int g, r0, nrows;
  if (!tc_resolve(pm, s_tab, s_yo, blockIdx.x, CH, &g, &r0, &nrows)) return;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  if (tid == 0) {
    for (int q = 0; q < kWgStages; q++) mbar_init(smem_u32(&bars[q]), 1);
    fence_barrier_init();
  }
  if (K < MA) {   // zero the padded feature blocks of every stage once
    for (int q = 0; q < kWgStages; q++)
      for (int i = tid; i < (int)((MA - K) / 32 * BLK / 16); i += 128)
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(
                         base + q * STAGE + (K / 32) * BLK + i * 16),
                     "r"(0));
  }
  // X row of every row of the chunk, resolved once up front (the dependent
  // y_src -> gather_ids loads would otherwise stall every stage)
  __shared__ int s_xrow[kCHT];
  const bool direct = Xm != nullptr;
  for (int base = tid; base < nrows; base += 8 * 128) {    // 8 dependent chains in flight
    int xr[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int i = base + u * 128;
      xr[u] = i < nrows ? (int)tc_a_row(pm, rel_y_off, y_src, gather_ids, g, r0 + i, direct) : 0;
    }
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (base + u * 128 < nrows) s_xrow[base + u * 128] = xr[u];
  }
  const float* Ab = (direct && g < pm.R) ? Xm : X;
  if (warp == 0) tmem_alloc(smem_u32(&tmem_slot), D);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  // B rows: dY of the relation (project-first) or, aggregate-first, the
  // gradient G of the relation's destination type (Z_r = Xagg_r W_r feeds
  // H_t(r) directly); root groups: G of the type
  const float* Bbase = g < pm.R ? (direct ? G + (long long)pm.type_dst_off[pm.rel_dst[g]] * D
                                          : dY + (long long)rel_y_off[g] * D)
                                : G + (long long)pm.type_dst_off[g - pm.R] * D;
  const int NST = (nrows + 31) / 32;

  auto load = [&](int c, int st) {
    const uint32_t sa = base + st * STAGE, sb = sa + A_STAGE;
#pragma unroll
    for (int q = 0; q < 32 * K / 4 / 128; q++) {
      const int i = tid + 128 * q;
      const int row = i / (K / 4), f = (i % (K / 4)) * 4;
      const int rr = c * 32 + row;
      const float* src = Ab;
      uint32_t nb = 0;
      if (rr < nrows) {
        src = Ab + (long long)s_xrow[rr] * K + f;
        nb = 16;
      }
      cp_async16(sa + (f >> 5) * BLK + (row >> 2) * 512 + sw128b32_off(row, (f & 31) * 4), src, nb);
    }
#pragma unroll
    for (int q = 0; q < 32 * D / 4 / 128; q++) {
      const int i = tid + 128 * q;
      const int row = i / (D / 4), f = (i % (D / 4)) * 4;
      const int rr = c * 32 + row;
      const float* src = Bbase;
      uint32_t nb = 0;
      if (rr < nrows) {
        src = Bbase + (long long)(r0 + rr) * D + f;
        nb = 16;
      }
      cp_async16(sb + (f >> 5) * BLK + (row >> 2) * 512 + sw128b32_off(row, (f & 31) * 4), src, nb);
    }
    cp_async_commit();
  };

  for (int c = 0; c < kWgStages - 1; c++) {
    if (c < NST) load(c, c);
    else cp_async_commit();
  }
  for (int c = 0; c < NST; c++) {
    const int st = c % kWgStages;
    const int nxt = c + kWgStages - 1;
    if (nxt < NST) {
      const int ns = nxt % kWgStages;
      if (nxt >= kWgStages) mbar_wait(smem_u32(&bars[ns]), ((nxt / kWgStages) - 1) & 1);
      load(nxt, ns);
    } else {
      cp_async_commit();
    }
    cp_async_wait<kWgStages - 1>();
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t sa = base + st * STAGE, sb = sa + A_STAGE;
#pragma unroll
      for (int k = 0; k < 4; k++)
        mma_tf32(tmem, sw128b32_desc(sa + k * 1024, BLK, 512), sw128b32_desc(sb + k * 1024, BLK, 512),
                 IDESC, (c | k) ? 1u : 0u);
      mma_commit(smem_u32(&bars[st]));
    }
    __syncwarp();
  }
  {
    const int c = NST - 1;
    mbar_wait(smem_u32(&bars[c % kWgStages]), (c / kWgStages) & 1);
    tc_fence_after();
  }
  // epilogue: TMEM lane = feature k (row of dW), columns = d
  const int k = warp * 32 + lane;
  float* P = partial + (long long)blockIdx.x * K * D + (long long)k * D;
#pragma unroll
  for (int c0 = 0; c0 < D; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
    if (k < K) {
      float4* o = reinterpret_cast<float4*>(P + c0);
      o[0] = make_float4(v[0], v[1], v[2], v[3]);
      o[1] = make_float4(v[4], v[5], v[6], v[7]);
      o[2] = make_float4(v[8], v[9], v[10], v[11]);
      o[3] = make_float4(v[12], v[13], v[14], v[15]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, D);
}

template <int K, int D, int KN>
static constexpr int dgrad_smem(int st) { return st * (128 * 128 + KN * 128) + 1024; }
template <int K, int D>
static constexpr int wgrad_smem() { return kWgStages * (4 * 4096 + (D / 32) * 4096) + 1024; }

// Pipeline depth per variant: a K = 128 layer splits the output features
// over two CTAs (KN = 64; 2 CTAs per SM need <= 4 stages of 24 KB), a K = 64
// layer keeps one CTA per tile with 6 producer warps / 6 stages.  Measured:
// IMDB inner-layer input gradient 23.4 -> 19.4 us with the split, mag
// unchanged; Freebase (K = 64) 23.4 -> 21.8 us with 6 stages.
template <int K, int D, int KN>
static void launch_dgrad(const DgradMeta& dm, int max_out, const int* slot_y, const float* dY,
                         const float* G, const float* W_rel, const float* W_root, float* dX,
                         cudaStream_t s) {
  constexpr int ST = (K / KN > 1) ? 4 : kDgStages, PR = (K / KN > 1) ? 4 : kDgProd;
  const int smem = dgrad_smem<K, D, KN>(ST) + max_out * 128 * 4;
  set_max_smem((const void*)k_dgrad_tc<K, D, KN, ST, PR>, smem);
  const unsigned grid = (unsigned)dm.tile_off[dm.T] * (K / KN);
  HF_LAUNCH((k_dgrad_tc<K, D, KN, ST, PR>), grid, (PR + 1) * 32, smem, s, dm, slot_y, dY, G,
            W_rel, W_root, dX, max_out);
}

hifuse_status dgrad_tc_launch(const DgradMeta& dm, int K, int D, const int* slot_y,
                              const float* dY, const float* G, const float* W_rel,
                              const float* W_root, float* dX, cudaStream_t s, long long dy_rows,
                              int R) {
  int max_out = 0;
  for (int t = 0; t < dm.T; t++) max_out = std::max(max_out, dm.out_off[t + 1] - dm.out_off[t]);
  if (max_out > 128) return HIFUSE_ERR_UNSUPPORTED;
  // K = 128: two CTAs per 128-row tile, 64 output features each (launch_dgrad)
  if (K == 128 && D == 128) launch_dgrad<128, 128, 64>(dm, max_out, slot_y, dY, G, W_rel, W_root, dX, s);
  else if (K == 128 && D == 64) launch_dgrad<128, 64, 64>(dm, max_out, slot_y, dY, G, W_rel, W_root, dX, s);
  else if (K == 64 && D == 128) launch_dgrad<64, 128, 64>(dm, max_out, slot_y, dY, G, W_rel, W_root, dX, s);
  else launch_dgrad<64, 64, 64>(dm, max_out, slot_y, dY, G, W_rel, W_root, dX, s);
  return HIFUSE_OK;
}

hifuse_status wgrad_tc_launch(const LayerMeta& m, const ProjMeta& pm, int K, int D, int CH,
                              const int* chunk_off, const int* rel_y_off, const int* y_src,
                              const int* gather_ids, const float* X, const float* dY,
                              const float* G, float* partial, unsigned grid, cudaStream_t s,
                              const float* Xm) {
  (void)m;
  {
    set_max_smem((const void*)k_wgrad_tc<128, 128>, wgrad_smem<128, 128>());
    set_max_smem((const void*)k_wgrad_tc<128, 64>, wgrad_smem<128, 64>());
    set_max_smem((const void*)k_wgrad_tc<64, 128>, wgrad_smem<64, 128>());
    set_max_smem((const void*)k_wgrad_tc<64, 64>, wgrad_smem<64, 64>());
  }
#define HF_WG(KK, DD)                                                                          \
  HF_LAUNCH((k_wgrad_tc<KK, DD>), grid, 128, (wgrad_smem<KK, DD>()), s, pm, CH, chunk_off,     \
            rel_y_off, y_src, gather_ids, X, dY, G, partial, Xm)
  if (K == 128 && D == 128) HF_WG(128, 128);
  else if (K == 128 && D == 64) HF_WG(128, 64);
  else if (K == 64 && D == 128) HF_WG(64, 128);
  else HF_WG(64, 64);
#undef HF_WG
  return HIFUSE_OK;
}

}  // namespace hf

namespace hf {

// ------------------------------------------------ persistent forward GEMM ----
// Two CTAs per SM, warp-specialised (the canonical Blackwell structure):
//   warps 0-3  producers: per 128-B K chunk, gather the tile's 128 A rows
//              (coalesced: one warp instruction = 4 rows x 128 B) into the
//              128B-swizzled K-major layout, and load the 32 x D slice of W_g
//              straight from its [K][D] storage as an MN-major operand
//              (SWIZZLE_128B_BASE32B) -- no transposed weight copy; a thread
//              signals a stage `full` kLag chunks later (cp.async groups retire
//              in order), after fence.proxy.async;
//   warp 8     one elected thread issues 4 tcgen05.mma (M=128, N=D, K=8) per
//              chunk into one of two TMEM accumulators, commits the stage's
//              `empty` barrier and, after a tile's last chunk, `tfull`;
//   warps 4-7  epilogue: tcgen05.ld (warp w reads TMEM lanes 32(w%4)..),
//              16-column slices staged in shared memory and written back as
//              8 rows x 64 contiguous bytes per instruction, then `tempty`.
// The tile table (128-row tiles per group) is built in shared memory from
// rel_y_off at kernel start.
#ifndef HF_F_STAGES
#define HF_F_STAGES 3
#endif
#ifndef HF_F_LAG
#define HF_F_LAG 2
#endif
#ifndef HF_F_CTAS
#define HF_F_CTAS 2
#endif
static constexpr int kFStages = HF_F_STAGES;
static constexpr int kLag = HF_F_LAG;
static constexpr int kFwdCtas = HF_F_CTAS;
static_assert(kLag < kFStages, "cp.async lag below the stage count");
// The fused fusion GEMM of the aggregate-first layers (k_fuse_gemm_tcp) has
// one 128-row tile per CTA (fewer tiles than SMs on every workload) and a long
// K loop ((1 + R_in) K): one CTA per SM with 4 stages beats two with 3
// (measured, mag: 16.8 -> 14.7 us); the per-relation projection, with many
// tiles per CTA, keeps two CTAs per SM (mag project-first: 83 vs 100-108 us
// with 1 CTA).
#ifndef HF_G_STAGES
#define HF_G_STAGES 4
#endif
static constexpr int kGStages = HF_G_STAGES;
#ifndef HF_G_LAG
#define HF_G_LAG 2
#endif
static constexpr int kGLag = HF_G_LAG;
static constexpr int kGCtas = 1;
static_assert(kGLag < kGStages, "cp.async lag below the stage count");

// Tiles (or chunks) of `step` rows per group -> s_tab[0..G], one warp.
__device__ __forceinline__ void group_table_warp(const ProjMeta& pm, const int* s_yoff, int step,
                                                 int* s_tab, int lane) {
  const int G = pm.R + pm.T;
  int carry = 0;
  for (int base = 0; base < G; base += 32) {
    const int g = base + lane;
    int rows = 0;
    if (g < pm.R) rows = s_yoff[g + 1] - s_yoff[g];
    else if (g < G && pm.has_root) rows = pm.n_dst[g - pm.R];
    const int t = (rows + step - 1) / step;
    int inc = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += n;
    }
    if (g < G) s_tab[g] = carry + inc - t;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) s_tab[G] = carry;
}

// BF16 (HIFUSE_PREC_BF16): the operands are rounded to bf16 (RN-even) on the
// way into shared memory -- A by the producer threads (fp32 X loads, cvt,
// st.shared into the same 128B-swizzled K-major layout, 64 bf16 per 128-byte
// row), B from Wt, W_g^T pre-rounded to bf16 [D][K] by k_w_bf16t (K-major,
// cp.async) -- and tcgen05.mma kind::f16 (K = 16 per instruction) accumulates
// in fp32.  Everything else (stages, barriers, epilogue) is shared.
// YB: the relation groups' rows (Y) are stored as bf16 (RN-even) into Yb
// (NEXT(3) byte diet: half the Y write and half the aggregation's gather);
// the root rows R0 stay fp32.
template <int K, int D, bool BF, bool YB>
__global__ void __launch_bounds__(288, kFwdCtas)
k_proj_fwd_tcp(ProjMeta pm, const int* __restrict__ rel_y_off, const int* __restrict__ y_src,
               const int* __restrict__ gather_ids, const float* __restrict__ X,
               const float* __restrict__ W_rel, const float* __restrict__ W_root,
               float* __restrict__ Y, float* __restrict__ R0, const float* __restrict__ att,
               float* __restrict__ s_src, int H, const float* __restrict__ Xm,
               const uint16_t* __restrict__ Wt, uint16_t* __restrict__ Yb) {
  HF_PDL_ENTRY();
  constexpr int BM = 128, KC = BF ? 64 : 32, NC = K / KC;   // K elements per 128-byte row
  constexpr uint32_t A_STAGE = BM * 128, B_BLK = 32 * 128, B_STAGE = (D / 32) * B_BLK;
  constexpr uint32_t STAGE = A_STAGE + B_STAGE;
  constexpr uint32_t IDESC = BF ? idesc_bf16(BM, D, 0, 0)    // A, B K-major
                                : idesc_tf32(BM, D, 0, 1);   // A K-major, B MN-major
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[kFStages], empty[kFStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  __shared__ int s_tile[HF_MAX_R + HF_MAX_T + 1], s_yoff[HF_MAX_R + 1];
  __shared__ __align__(16) float stage_ep[4 * 32 * 20];     // epilogue staging
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  for (int i = tid; i <= pm.R; i += blockDim.x) s_yoff[i] = rel_y_off[i];
  if (tid == 0) {
    for (int q = 0; q < kFStages; q++) {
      mbar_init(smem_u32(&full[q]), 128);
      mbar_init(smem_u32(&empty[q]), 1);
    }
    for (int q = 0; q < 2; q++) {
      mbar_init(smem_u32(&tfull[q]), 1);
      mbar_init(smem_u32(&tempty[q]), 128);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0) group_table_warp(pm, s_yoff, BM, s_tile, lane);
  if (warp == 8) tmem_alloc(smem_u32(&tmem_slot), 2 * D);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int ntiles = s_tile[pm.R + pm.T];

  if (warp < 4) {
    // ------------------------------------------------------------ producers
    // producer warp w owns tile rows [32w, 32w+32); lane l serves rows
    // 32w + 4i + l/8 (i = 0..7), 16-byte piece l%8 of every K chunk; the next
    // tile's row addresses are fetched one tile ahead.
    const int piece = lane & 7, rsub = lane >> 3;
    auto rows_of = [&](int t, int* g, const float** ap, uint32_t* nb) {
      int r0, nrows;
      tc_resolve(pm, s_tile, s_yoff, t, BM, g, &r0, &nrows);
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int row = warp * 32 + i * 4 + rsub;
        ap[i] = X;
        nb[i] = 0;
        if (row < nrows) {
          const float* Ab = (Xm && *g < pm.R) ? Xm : X;
          ap[i] = Ab + tc_a_row(pm, s_yoff, y_src, gather_ids, *g, r0 + row, Xm != nullptr) * K;
          nb[i] = 16;
        }
      }
    };
    int it = 0;
    int g = 0;
    const float* ap[8];
    uint32_t nb[8];
#pragma unroll
    for (int i = 0; i < 8; i++) { ap[i] = X; nb[i] = 0; }
    if ((int)blockIdx.x < ntiles) rows_of(blockIdx.x, &g, ap, nb);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int ng = 0;
      const float* nap[8];
      uint32_t nnb[8];
#pragma unroll
      for (int i = 0; i < 8; i++) { nap[i] = X; nnb[i] = 0; }
      if (t + (int)gridDim.x < ntiles) rows_of(t + gridDim.x, &ng, nap, nnb);
      const float* Wg = g < pm.R ? W_rel + (long long)g * K * D : W_root + (long long)(g - pm.R) * K * D;
      for (int c = 0; c < NC; c++, it++) {
        const int s = it % kFStages;
        if constexpr (BF) {
          // A: 8 fp32 of each of the lane's 8 rows, loaded before the stage
          // wait (in flight meanwhile), rounded to bf16 and stored as one
          // 16-byte piece of the swizzled row
          // (two halves of 4 rows: 8 float4 in flight per lane, no spills)
          const uint32_t sa = base + s * STAGE, sb = sa + A_STAGE;
#pragma unroll
          for (int hh = 0; hh < 2; hh++) {
            float4 xa[4][2];
#pragma unroll
            for (int i = 0; i < 4; i++) {
              const int ii = hh * 4 + i;
              const float4* src = reinterpret_cast<const float4*>(ap[ii] + c * 64 + piece * 8);
              xa[i][0] = nb[ii] ? __ldg(src) : make_float4(0.f, 0.f, 0.f, 0.f);
              xa[i][1] = nb[ii] ? __ldg(src + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (hh == 0 && it >= kFStages) mbar_wait(smem_u32(&empty[s]), ((it / kFStages) - 1) & 1);
#pragma unroll
            for (int i = 0; i < 4; i++) {
              const int row = warp * 32 + (hh * 4 + i) * 4 + rsub;
              st_shared_bf16x8(sa + sw128_off(row, piece), xa[i][0], xa[i][1]);
            }
          }
          // B: Wt[g] rows n = 0 .. D-1, K elements 64c .. 64c+63 (K-major)
          const uint16_t* Wtg = Wt + (long long)g * D * K;
#pragma unroll
          for (int q = 0; q < D * 8 / 128; q++) {
            const int i = tid + 128 * q;
            const int n = i >> 3, pc = i & 7;
            cp_async16(sb + sw128_off(n, pc), Wtg + (long long)n * K + c * 64 + pc * 8, 16);
          }
        } else {
          if (it >= kFStages) mbar_wait(smem_u32(&empty[s]), ((it / kFStages) - 1) & 1);
          const uint32_t sa = base + s * STAGE, sb = sa + A_STAGE;
#pragma unroll
          for (int i = 0; i < 8; i++) {
            const int row = warp * 32 + i * 4 + rsub;
            cp_async16(sa + sw128_off(row, piece), ap[i] + c * 32 + piece * 4, nb[i]);
          }
          // B: rows k = 32c .. 32c+31 of W_g, D floats each, MN-major atoms
#pragma unroll
          for (int q = 0; q < 32 * D / 4 / 128; q++) {
            const int i = tid + 128 * q;
            const int kr = i / (D / 4), n = (i % (D / 4)) * 4;
            cp_async16(sb + (n >> 5) * B_BLK + (kr >> 2) * 512 + sw128b32_off(kr, (n & 31) * 4),
                       Wg + (long long)(c * 32 + kr) * D + n, 16);
          }
        }
        cp_async_commit();
        if (it >= kLag) {
          cp_async_wait<kLag>();
          fence_proxy_async();
          mbar_arrive(smem_u32(&full[(it - kLag) % kFStages]));
        }
      }
      g = ng;
#pragma unroll
      for (int i = 0; i < 8; i++) { ap[i] = nap[i]; nb[i] = nnb[i]; }
    }
    cp_async_wait<0>();
    fence_proxy_async();
    for (int j = it - kLag < 0 ? 0 : it - kLag; j < it; j++) mbar_arrive(smem_u32(&full[j % kFStages]));
  } else if (warp < 8) {
    // ------------------------------------------------------------- epilogue
    const int q = warp - 4;
    int tc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, tc++) {
      const int acc = tc & 1;
      int g, r0, nrows;
      tc_resolve(pm, s_tile, s_yoff, t, BM, &g, &r0, &nrows);
      mbar_wait(smem_u32(&tfull[acc]), (tc >> 1) & 1);
      tc_fence_after();
      float* out = g < pm.R ? Y + (long long)s_yoff[g] * D
                            : R0 + (long long)pm.type_dst_off[g - pm.R] * D;
      float* st = stage_ep + q * (32 * 20);
      // RGAT source scores fused here: s_src[u,h] = <Y[u, head h], a_src[r, head h]>
      const bool scores = att != nullptr && g < pm.R;
      const int dh = scores ? D / H : 0;
      const float* asrc = scores ? att + (long long)g * 2 * D : nullptr;
      float* srow = scores ? s_src + (long long)(s_yoff[g] + r0 + q * 32 + lane) * H : nullptr;
      const bool row_ok = q * 32 + lane < nrows;
      float sacc = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + (uint32_t)(acc * D) + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
        if (scores) {
          float qs[4];
#pragma unroll
          for (int qq = 0; qq < 4; qq++) {
            const float4 a4 = __ldg(reinterpret_cast<const float4*>(asrc + c0) + qq);
            qs[qq] = v[4 * qq] * a4.x + v[4 * qq + 1] * a4.y + v[4 * qq + 2] * a4.z + v[4 * qq + 3] * a4.w;
          }
          if (row_ok) {
            if (dh == 4) {
#pragma unroll
              for (int qq = 0; qq < 4; qq++) srow[c0 / 4 + qq] = qs[qq];
            } else if (dh == 8) {
              srow[c0 / 8] = qs[0] + qs[1];
              srow[c0 / 8 + 1] = qs[2] + qs[3];
            } else if (dh == 16) {
              srow[c0 / 16] = (qs[0] + qs[1]) + (qs[2] + qs[3]);
            }
          }
          if (dh >= 32) {
            sacc += (qs[0] + qs[1]) + (qs[2] + qs[3]);
            if ((c0 + 16) % dh == 0) {
              if (row_ok) srow[c0 / dh] = sacc;
              sacc = 0.f;
            }
          }
        }
#pragma unroll
        for (int jj = 0; jj < 4; jj++)
          *reinterpret_cast<float4*>(st + lane * 20 + 4 * jj) =
              make_float4(v[4 * jj], v[4 * jj + 1], v[4 * jj + 2], v[4 * jj + 3]);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int rr = i * 8 + (lane >> 2), ch = lane & 3;
          const int row = q * 32 + rr;
          const float4 x = *reinterpret_cast<const float4*>(st + rr * 20 + 4 * ch);
          if (YB && g < pm.R) {
            if (row < nrows) {
              uint2 w;
              asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w.x) : "f"(x.y), "f"(x.x));
              asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w.y) : "f"(x.w), "f"(x.z));
              *reinterpret_cast<uint2*>(Yb + (long long)(s_yoff[g] + r0 + row) * D + c0 + 4 * ch) = w;
            }
          } else if (row < nrows) {
            *reinterpret_cast<float4*>(out + (long long)(r0 + row) * D + c0 + 4 * ch) = x;
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(smem_u32(&tempty[acc]));
    }
  } else if (lane == 0) {
    // ------------------------------------------------------------------ MMA
    int it = 0, tc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, tc++) {
      const int acc = tc & 1;
      if (tc >= 2) mbar_wait(smem_u32(&tempty[acc]), ((tc >> 1) - 1) & 1);
      tc_fence_after();
      for (int c = 0; c < NC; c++, it++) {
        const int s = it % kFStages;
        mbar_wait(smem_u32(&full[s]), (it / kFStages) & 1);
        tc_fence_after();
        const uint32_t sa = base + s * STAGE, sb = sa + A_STAGE;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          if constexpr (BF)      // K = 16 bf16 = 32 bytes per MMA along both K-major rows
            mma_f16(tmem + (uint32_t)(acc * D), sw128_desc(sa + k * 32, 16, 1024),
                    sw128_desc(sb + k * 32, 16, 1024), IDESC, (c | k) ? 1u : 0u);
          else
            mma_tf32(tmem + (uint32_t)(acc * D), sw128_desc(sa + k * 32, 16, 1024),
                     sw128b32_desc(sb + k * 1024, B_BLK, 512), IDESC, (c | k) ? 1u : 0u);
        }
        mma_commit(smem_u32(&empty[s]));
      }
      mma_commit(smem_u32(&tfull[acc]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc(tmem, 2 * D);
}

// Wt[g][n][k] = bf16_rn(W_g[k][n]) for the R relation weights then the T root
// weights (transposed to K-major, the B layout of the BF16 projection).
__global__ void k_w_bf16t(int R, int T, int K, int D, const float* __restrict__ W_rel,
                          const float* __restrict__ W_root, uint16_t* __restrict__ Wt) {
  HF_PDL_ENTRY();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (long long)K * D;
  if (i >= (R + T) * per) return;
  const int g = (int)(i / per);
  const int n = (int)(i % per) / K, k = (int)(i % per) % K;
  const float w = g < R ? W_rel[(long long)g * per + (long long)k * D + n]
                        : W_root[(long long)(g - R) * per + (long long)k * D + n];
  Wt[i] = __bfloat16_as_ushort(__float2bfloat16_rn(w));
}

// ------------------------------------------- fused fusion GEMM (NEXT(3)) ----
// Aggregate-first RGCN input layer, projection + semantic fusion as ONE
// tcgen05 GEMM per destination type (PAPER.md lines
// 265-268, merging for memory efficiency and fewer kernels):
//   H_t[i] = act( [X_t[i] | Xagg_{r1}[i] | Xagg_{r2}[i] | ...]
//                 . [W_root,t ; W_r1 ; W_r2 ; ...] + b_t ),  r_j: t(r_j) = t,
// i.e. K = (1 + R_in(t)) * K_in, accumulated in one TMEM tile, bias and ReLU
// in the epilogue, H written once: no Z [rho, D] / R0 write and re-read, no
// separate fusion kernel.  Same warp specialisation, swizzles and stages as
// k_proj_fwd_tcp; the A rows of a K segment come from the feature store
// (root segment, through gather_ids) or from the aggregated rows
// Xagg[rel_row_off[r] + i]; the B chunks from W_root[t] / W_rel[r].
struct FuseGemmMeta {
  int T, R, has_root;
  int tile_off[HF_MAX_T + 1];      // 128-row tiles of each destination type
  int n_dst[HF_MAX_T];
  int type_src_off[HF_MAX_T + 1];
  int type_dst_off[HF_MAX_T + 1];
  int in_off[HF_MAX_T + 1];        // relations into type t: in_rel[in_off[t] .. in_off[t+1])
  int in_rel[HF_MAX_R];
  int rel_row_off[HF_MAX_R + 1];
};

template <int K, int D, bool RELU>
__global__ void __launch_bounds__(288, kGCtas)
k_fuse_gemm_tcp(FuseGemmMeta fm, const int* __restrict__ gather_ids, const float* __restrict__ X,
                const float* __restrict__ Xm, const float* __restrict__ W_rel,
                const float* __restrict__ W_root, const float* __restrict__ bias,
                float* __restrict__ H) {
  HF_PDL_ENTRY();
  constexpr int BM = 128, NCS = K / 32;                      // chunks per K segment
  constexpr uint32_t A_STAGE = BM * 128, B_BLK = 32 * 128, B_STAGE = (D / 32) * B_BLK;
  constexpr uint32_t STAGE = A_STAGE + B_STAGE;
  constexpr uint32_t IDESC = idesc_tf32(BM, D, 0, 1);      // A K-major, B MN-major
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[kGStages], empty[kGStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(16) float stage_ep[4 * 32 * 20];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  if (tid == 0) {
    for (int q = 0; q < kGStages; q++) {
      mbar_init(smem_u32(&full[q]), 128);
      mbar_init(smem_u32(&empty[q]), 1);
    }
    for (int q = 0; q < 2; q++) {
      mbar_init(smem_u32(&tfull[q]), 1);
      mbar_init(smem_u32(&tempty[q]), 128);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 8) tmem_alloc(smem_u32(&tmem_slot), 2 * D);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int ntiles = fm.tile_off[fm.T];
  // tile -> (type, first row, rows, K segments)
  auto resolve = [&](int t, int* ty, int* r0, int* nrows, int* nseg) {
    int lo = 0, hi = fm.T;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (fm.tile_off[mid] <= t) lo = mid; else hi = mid;
    }
    *ty = lo;
    *r0 = (t - fm.tile_off[lo]) * BM;
    *nrows = min(BM, fm.n_dst[lo] - *r0);
    *nseg = fm.has_root + fm.in_off[lo + 1] - fm.in_off[lo];
  };
  if (warp < 4) {
    // ------------------------------------------------------------ producers
    const int piece = lane & 7, rsub = lane >> 3;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int ty, r0, nrows, nseg;
      resolve(t, &ty, &r0, &nrows, &nseg);
      for (int sg = 0; sg < nseg; sg++) {
        // segment sg: root (sg == 0 with a root term) or relation in_rel[...]
        const bool root = fm.has_root && sg == 0;
        const int r = root ? -1 : fm.in_rel[fm.in_off[ty] + sg - fm.has_root];
        const float* Wg = root ? W_root + (long long)ty * K * D : W_rel + (long long)r * K * D;
        const float* ap[8];
        uint32_t nb[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const int row = warp * 32 + i * 4 + rsub;
          ap[i] = Xm;
          nb[i] = 0;
          if (row < nrows) {
            if (root) {
              const int x = fm.type_src_off[ty] + r0 + row;     // destinations: source prefix
              ap[i] = X + (long long)(gather_ids ? gather_ids[x] : x) * K;
            } else {
              ap[i] = Xm + (long long)(fm.rel_row_off[r] + r0 + row) * K;
            }
            nb[i] = 16;
          }
        }
        for (int c = 0; c < NCS; c++, it++) {
          const int s = it % kGStages;
          if (it >= kGStages) mbar_wait(smem_u32(&empty[s]), ((it / kGStages) - 1) & 1);
          const uint32_t sa = base + s * STAGE, sb = sa + A_STAGE;
#pragma unroll
          for (int i = 0; i < 8; i++) {
            const int row = warp * 32 + i * 4 + rsub;
            cp_async16(sa + sw128_off(row, piece), ap[i] + c * 32 + piece * 4, nb[i]);
          }
#pragma unroll
          for (int q = 0; q < 32 * D / 4 / 128; q++) {
            const int i = tid + 128 * q;
            const int kr = i / (D / 4), n = (i % (D / 4)) * 4;
            cp_async16(sb + (n >> 5) * B_BLK + (kr >> 2) * 512 + sw128b32_off(kr, (n & 31) * 4),
                       Wg + (long long)(c * 32 + kr) * D + n, 16);
          }
          cp_async_commit();
          if (it >= kGLag) {
            cp_async_wait<kGLag>();
            fence_proxy_async();
            mbar_arrive(smem_u32(&full[(it - kGLag) % kGStages]));
          }
        }
      }
    }
    cp_async_wait<0>();
    fence_proxy_async();
    for (int j = it - kGLag < 0 ? 0 : it - kGLag; j < it; j++) mbar_arrive(smem_u32(&full[j % kGStages]));
  } else if (warp < 8) {
    // ------------------------------------------------------------- epilogue
    const int q = warp - 4;
    int tc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, tc++) {
      const int acc = tc & 1;
      int ty, r0, nrows, nseg;
      resolve(t, &ty, &r0, &nrows, &nseg);
      mbar_wait(smem_u32(&tfull[acc]), (tc >> 1) & 1);
      tc_fence_after();
      float* out = H + (long long)(fm.type_dst_off[ty] + r0) * D;
      const float* bt = bias ? bias + (long long)ty * D : nullptr;
      float* st = stage_ep + q * (32 * 20);
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + (uint32_t)(acc * D) + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
        if (nseg == 0) {
#pragma unroll
          for (int jj = 0; jj < 16; jj++) v[jj] = 0.f;    // no term at all: act(b)
        }
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
          float4 b4 = bt ? __ldg(reinterpret_cast<const float4*>(bt + c0) + jj)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
          float4 o4 = make_float4(v[4 * jj] + b4.x, v[4 * jj + 1] + b4.y, v[4 * jj + 2] + b4.z,
                                  v[4 * jj + 3] + b4.w);
          if (RELU) {
            o4.x = fmaxf(o4.x, 0.f); o4.y = fmaxf(o4.y, 0.f);
            o4.z = fmaxf(o4.z, 0.f); o4.w = fmaxf(o4.w, 0.f);
          }
          *reinterpret_cast<float4*>(st + lane * 20 + 4 * jj) = o4;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int rr = i * 8 + (lane >> 2), ch = lane & 3;
          const int row = q * 32 + rr;
          const float4 x = *reinterpret_cast<const float4*>(st + rr * 20 + 4 * ch);
          if (row < nrows) *reinterpret_cast<float4*>(out + (long long)row * D + c0 + 4 * ch) = x;
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(smem_u32(&tempty[acc]));
    }
  } else if (lane == 0) {
    // ------------------------------------------------------------------ MMA
    int it = 0, tc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, tc++) {
      const int acc = tc & 1;
      int ty, r0, nrows, nseg;
      resolve(t, &ty, &r0, &nrows, &nseg);
      if (tc >= 2) mbar_wait(smem_u32(&tempty[acc]), ((tc >> 1) - 1) & 1);
      tc_fence_after();
      const int nc = nseg * NCS;
      for (int c = 0; c < nc; c++, it++) {
        const int s = it % kGStages;
        mbar_wait(smem_u32(&full[s]), (it / kGStages) & 1);
        tc_fence_after();
        const uint32_t sa = base + s * STAGE, sb = sa + A_STAGE;
#pragma unroll
        for (int k = 0; k < 4; k++)
          mma_tf32(tmem + (uint32_t)(acc * D), sw128_desc(sa + k * 32, 16, 1024),
                   sw128b32_desc(sb + k * 1024, B_BLK, 512), IDESC, (c | k) ? 1u : 0u);
        mma_commit(smem_u32(&empty[s]));
      }
      mma_commit(smem_u32(&tfull[acc]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc(tmem, 2 * D);
}

template <int K, int D>
static constexpr int fwdp_smem() { return kFStages * (128 * 128 + D * 128) + 1024; }
template <int K, int D>
static constexpr int fuseg_smem() { return kGStages * (128 * 128 + D * 128) + 1024; }

template <int K, int D, bool BF, bool YB>
static void launch_tcp(const ProjMeta& pm, const int* rel_off, const int* y_src,
                       const int* gather_ids, const float* X, const float* Xm,
                       const float* W_rel, const float* W_root, float* Y, float* R0,
                       const float* att, float* s_src, int H, const uint16_t* Wt,
                       uint16_t* Yb, cudaStream_t s) {
  set_max_smem(reinterpret_cast<const void*>(&k_proj_fwd_tcp<K, D, BF, YB>), fwdp_smem<K, D>());
  HF_LAUNCH((k_proj_fwd_tcp<K, D, BF, YB>), sm_count() * kFwdCtas, 288, (fwdp_smem<K, D>()), s,
            pm, rel_off, y_src, gather_ids, X, W_rel, W_root, Y, R0, att, s_src, H, Xm, Wt, Yb);
}

template <int K, int D, bool RELU>
static void launch_fuse_gemm(const FuseGemmMeta& fm, const int* gid, const float* X,
                             const float* Xm, const float* W_rel, const float* W_root,
                             const float* bias, float* H, cudaStream_t s) {
  set_max_smem(reinterpret_cast<const void*>(&k_fuse_gemm_tcp<K, D, RELU>), fuseg_smem<K, D>());
  HF_LAUNCH((k_fuse_gemm_tcp<K, D, RELU>), sm_count() * kGCtas, 288, (fuseg_smem<K, D>()), s, fm,
            gid, X, Xm, W_rel, W_root, bias, H);
}

hifuse_status fuse_gemm_launch(const LayerMeta& m, bool has_root, int K, int D, bool relu,
                               const int* gid, const float* X, const float* Xm,
                               const float* W_rel, const float* W_root, const float* bias,
                               float* H, cudaStream_t s) {
  FuseGemmMeta fm;
  fm.T = m.T;
  fm.R = m.R;
  fm.has_root = has_root ? 1 : 0;
  int tiles = 0, k = 0;
  for (int t = 0; t < m.T; t++) {
    fm.tile_off[t] = tiles;
    tiles += (m.n_dst[t] + 127) / 128;
    fm.n_dst[t] = m.n_dst[t];
    fm.in_off[t] = k;
    for (int r = 0; r < m.R; r++)
      if (m.rel_dst[r] == t) fm.in_rel[k++] = r;
  }
  fm.tile_off[m.T] = tiles;
  fm.in_off[m.T] = k;
  for (int t = 0; t <= m.T; t++) {
    fm.type_src_off[t] = m.type_src_off[t];
    fm.type_dst_off[t] = m.type_dst_off[t];
  }
  for (int r = 0; r <= m.R; r++) fm.rel_row_off[r] = m.rel_row_off[r];
  if (tiles == 0) return HIFUSE_OK;
#define HF_FG(KK, DD)                                                                          \
  if (relu) launch_fuse_gemm<KK, DD, true>(fm, gid, X, Xm, W_rel, W_root, bias, H, s);         \
  else launch_fuse_gemm<KK, DD, false>(fm, gid, X, Xm, W_rel, W_root, bias, H, s)
  if (K == 128 && D == 128) { HF_FG(128, 128); }
  else if (K == 128 && D == 64) { HF_FG(128, 64); }
  else if (K == 64 && D == 128) { HF_FG(64, 128); }
  else { HF_FG(64, 64); }
#undef HF_FG
  return HIFUSE_OK;
}

hifuse_status project_tcp_launch(const LayerMeta& m, const ProjMeta& pm, int K, int D,
                                 const int* rel_off, const int* y_src, const float* X,
                                 const float* Xm, const int* gather_ids, const float* W_rel,
                                 const float* W_root, float* Y, float* R0, const float* att,
                                 float* s_src, int H, cudaStream_t s, uint16_t* Wt_bf16,
                                 uint16_t* Yb) {
  if (Wt_bf16) {             // BF16 operands: round + transpose the weights first
    const int G = m.R + (W_root ? m.T : 0);
    HF_LAUNCH(k_w_bf16t, ceil_div((long long)G * K * D, 256), 256, 0, s, m.R, W_root ? m.T : 0, K,
              D, W_rel, W_root, Wt_bf16);
  }
#define HF_TCP2(KK, DD, YBB)                                                                    \
  if (Wt_bf16)                                                                                 \
    launch_tcp<KK, DD, true, YBB>(pm, rel_off, y_src, gather_ids, X, Xm, W_rel, W_root, Y, R0,  \
                                  att, s_src, H, Wt_bf16, Yb, s);                               \
  else                                                                                         \
    launch_tcp<KK, DD, false, YBB>(pm, rel_off, y_src, gather_ids, X, Xm, W_rel, W_root, Y, R0, \
                                   att, s_src, H, nullptr, Yb, s)
#define HF_TCP(KK, DD)                                                                          \
  if (Yb) { HF_TCP2(KK, DD, true); } else { HF_TCP2(KK, DD, false); }
  if (K == 128 && D == 128) { HF_TCP(128, 128); }
  else if (K == 128 && D == 64) { HF_TCP(128, 64); }
  else if (K == 64 && D == 128) { HF_TCP(64, 128); }
  else { HF_TCP(64, 64); }
#undef HF_TCP
#undef HF_TCP2
  return HIFUSE_OK;
}

}  // namespace hf

// sample.cu -- GPU neighbour sampler (Fig. 2
// step (1), line 156; SPEC.md sample_batch S:L126-143).  include/hifuse.h
// documents the contract.  Per hop (innermost layer first), 7 kernels and two
// scans, independent of R and of the batch:
//   k_smp_mark_dst  destinations: gen[v] = stamp, loc[v] = local id
//   k_smp_pairs     warp per (destination, relation into its type): Floyd's
//                   uniform k-subset of the in-list (k = min(deg, fanout)),
//                   sorted; picks go to fixed slots; first sight of a new
//                   source vertex (atomicExch on gen) sets its bit in a
//                   per-type bitmap
//   k_smp_popc      popcount per bitmap word            -> scan: source ranks
//   [scan of per-pair counts]                           -> edge positions
//   k_smp_counts    n_src, n_dst, N; next hop's type offsets
//   k_smp_assign    new sources get n_dst + rank (ascending vertex id); the
//                   block's type-major source list (destinations first)
//   k_smp_edges     compaction of the slots into (src_local, dst_local, eid)
// Randomness: splitmix64 counter hash of (hop key, r, v, j): no RNG state.
#include <algorithm>
#include <cstring>
#include <vector>
#include "common.cuh"

namespace hf {

static constexpr int kMaxFan = 64;

// Padded (capacity) layout of one hop's block (hifuse_sample_blocks_padded):
// type t's sources start at off[t] (prefix of the per-type capacities), slots
// past the sampled ones hold -1 (gather id: the type's first row), edge
// positions [N, ecap) are null edges (edge_id -1).  on = 0: compact layout.
struct PadCaps {
  int on;
  int off[HF_MAX_T + 1];
  long long ecap;
};

struct SmpMeta {
  int T, R, Rmax;
  long long goff[HF_MAX_T + 1];       // prefix of |V_t|: state / feature-store offsets
  int wbase[HF_MAX_T + 1];            // bitmap word offset of type t
  int trel_off[HF_MAX_T + 1];         // relations into type t: trel[trel_off[t] .. +1)
  int trel[HF_MAX_R];
  int rel_src[HF_MAX_R];
  long long in_ptr_off[HF_MAX_R];
  long long count[HF_MAX_T];
};

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// uniform integer in [0, j] from the hash of (hk, r, v, j) (multiply-shift)
__device__ __forceinline__ int rand_upto(unsigned long long hk, int r, int v, int j) {
  unsigned long long h = mix64(mix64(mix64(hk ^ (unsigned long long)r) ^ (unsigned long long)v) ^
                               (unsigned long long)j);
  return (int)(((h >> 32) * (unsigned long long)(j + 1)) >> 32);
}

__device__ __forceinline__ int type_of(const int* fo, int T, int d) {
  int t = 0;
  while (t + 1 < T && fo[t + 1] <= d) t++;
  return t;
}

__global__ void k_smp_init(int T, int target, int B, int* __restrict__ fo) {
  HF_PDL_ENTRY();
  int t = threadIdx.x;
  if (t <= T) fo[t] = t <= target ? 0 : B;
}

__global__ void __launch_bounds__(256)
k_smp_mark_dst(SmpMeta m, const int* __restrict__ fo_d, const int* __restrict__ front,
               int* __restrict__ gen, int* __restrict__ loc, int stamp,
               const unsigned long long* __restrict__ d_ctl, int hop, int pad,
               int* __restrict__ status) {
  HF_PDL_ENTRY();
  __shared__ int fo[HF_MAX_T + 1];
  for (int i = threadIdx.x; i <= m.T; i += blockDim.x) fo[i] = fo_d[i];
  __syncthreads();
  if (d_ctl) stamp = (int)d_ctl[1] + hop;
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= fo[m.T]) return;
  const int t = type_of(fo, m.T, d);
  const int v = front[d];
  if (pad && v == -1) return;                     // padding slot of the previous hop
  if (v < 0 || v >= m.count[t]) {
    atomicOr(status, HIFUSE_ST_BAD_DST);
    return;
  }
  const long long g = m.goff[t] + v;
  gen[g] = stamp;
  loc[g] = d - fo[t];
}

// Warp per (destination, relation into its type) pair.  Floyd's picks are
// resolved in order, but the hashes are not sequential: lane i hashes step i
// (and i + 32), the recurrence then costs one shuffle and one ballot per
// step, with the selected in-list positions held one per lane (entries n and
// n + 32 in s0 / s1).  The positions are ranked (ascending in-list order) and
// each lane does the memory work of its picks -- in-list loads, first-sight
// atomicExch / bitmap atomicOr, slot stores -- so a pair's k picks cost one
// round trip.  Measured on ogbn-mag (us per hop, inner / outer): thread per
// pair with serial picks 56 / 56 (k dependent atomic round trips); warp per
// pair hashing every step on every lane 10 / 75 (32x redundant hashes);
// thread per pair + warp-cooperative picks 62 / 66 (32 dependent rounds).
constexpr int kSmpWarps = 8;

__global__ void __launch_bounds__(kSmpWarps * 32)
k_smp_pairs(SmpMeta m, const int* __restrict__ fo_d, const int* __restrict__ front, int P, int f,
            unsigned long long hk, const unsigned long long* __restrict__ d_ctl, int hop,
            const long long* __restrict__ in_ptr,
            const int* __restrict__ in_src, const long long* __restrict__ in_eid,
            int* __restrict__ gen, unsigned* __restrict__ bitmap, int stamp,
            int* __restrict__ slot_src, long long* __restrict__ slot_eid,
            int* __restrict__ pair_cnt) {
  HF_PDL_ENTRY();
  __shared__ int fo[HF_MAX_T + 1];
  __shared__ int sorted[kSmpWarps][kMaxFan];
  for (int i = threadIdx.x; i <= m.T; i += blockDim.x) fo[i] = fo_d[i];
  __syncthreads();
  if (d_ctl) {                       // key and stamp base from device memory
    hk = mix64(d_ctl[0] ^ (0x1000ull + (unsigned long long)hop));
    stamp = (int)d_ctl[1] + hop;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // grid-stride over the pairs of the actual frontier (fo[T] destinations;
  // the host bound P is the worst case: a grid over it spent most of its time
  // dispatching blocks that exit)
  const long long Pact = min((long long)P, (long long)fo[m.T] * m.Rmax);
  for (long long p = Pact + (long long)blockIdx.x * blockDim.x + threadIdx.x; p < P;
       p += (long long)gridDim.x * blockDim.x)
    pair_cnt[p] = 0;                                   // past the frontier (scanned over P)
  // Pairs of a warp: p, p + S, p + 2S, ...  The frontier vertex of the pair
  // two ahead and the in-list pointers of the next pair are loaded before the
  // current pair is processed, so its two dependent round trips (front ->
  // in_ptr) overlap the current pair's selection and atomics.
  const long long S = (long long)gridDim.x * kSmpWarps;
  struct PairA { int r, v; };                            // relation (-1: none), vertex
  struct PairB { long long base; int deg; };
  auto stage_a = [&](long long pp) -> PairA {
    PairA x{-1, 0};
    if (pp < Pact) {
      const int d = (int)(pp / m.Rmax), q = (int)(pp % m.Rmax);
      const int t = type_of(fo, m.T, d);
      if (q < m.trel_off[t + 1] - m.trel_off[t]) {
        const int v = front[d];
        if (v >= 0 && v < m.count[t]) { x.r = m.trel[m.trel_off[t] + q]; x.v = v; }
      }
    }
    return x;
  };
  auto stage_b = [&](const PairA& x) -> PairB {
    PairB y{0, 0};
    if (x.r >= 0) {
      const long long* ptr = in_ptr + m.in_ptr_off[x.r] + x.v;
      y.base = ptr[0];
      y.deg = (int)(ptr[1] - y.base);
    }
    return y;
  };
  long long p = (long long)blockIdx.x * kSmpWarps + w;
  PairA a0 = stage_a(p), a1 = stage_a(p + S);
  PairB b0 = stage_b(a0);
  for (; p < Pact; p += S) {
  const PairA a2 = stage_a(p + 2 * S);
  const PairB b1 = stage_b(a1);
  int k = 0;
  {
    if (a0.r >= 0) {
      const int r = a0.r, v = a0.v;
      const long long base = b0.base;
      const int deg = b0.deg;
      k = min(deg, f);
      int* srt = sorted[w];
      if (deg <= f) {                                  // every in-edge, in order
        for (int j = lane; j < k; j += 32) srt[j] = j;
      } else {
        // Floyd: for j = deg-k .. deg-1, c = U[0, j]; take c unless taken, else j
        const int j0 = deg - k;
        const int c0 = lane < k ? rand_upto(hk, r, v, j0 + lane) : 0;
        const int c1 = lane + 32 < k ? rand_upto(hk, r, v, j0 + lane + 32) : 0;
        int s0 = 0x7fffffff, s1 = 0x7fffffff;
        for (int i = 0; i < k; i++) {
          const int c = i < 32 ? __shfl_sync(0xffffffffu, c0, i)
                               : __shfl_sync(0xffffffffu, c1, i - 32);
          const bool taken = __any_sync(0xffffffffu, s0 == c || s1 == c);
          const int val = taken ? j0 + i : c;
          if (i == lane) s0 = val;
          else if (i == lane + 32) s1 = val;
        }
        // ascending in-list order: rank among the k (distinct) entries
        int r0 = 0, r1 = 0;
        const int na = k < 32 ? k : 32;
        for (int a = 0; a < na; a++) {
          const int x0 = __shfl_sync(0xffffffffu, s0, a);
          r0 += x0 < s0;
          r1 += x0 < s1;
        }
        if (k > 32)
          for (int a = 0; a < k - 32; a++) {
            const int x1 = __shfl_sync(0xffffffffu, s1, a);
            r0 += x1 < s0;
            r1 += x1 < s1;
          }
        if (lane < k) srt[r0] = s0;
        if (lane + 32 < k) srt[r1] = s1;
      }
      __syncwarp();
      const int s = m.rel_src[r];
      for (int j = lane; j < k; j += 32) {
        const long long e = base + srt[j];
        const int u = in_src[e];
        const long long id = in_eid[e];
        if (atomicExch(gen + m.goff[s] + u, stamp) != stamp)
          atomicOr(bitmap + m.wbase[s] + (u >> 5), 1u << (u & 31));
        slot_src[p * f + j] = u;
        slot_eid[p * f + j] = id;
      }
      __syncwarp();                                    // srt reused by the next pair
    }
  }
  if (lane == 0) pair_cnt[p] = k;
  a0 = a1; b0 = b1; a1 = a2;
  }
}

__global__ void k_smp_popc(const unsigned* __restrict__ bitmap, int W, int* __restrict__ wcnt) {
  HF_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < W) wcnt[i] = __popc(bitmap[i]);
}

__global__ void k_smp_counts(SmpMeta m, const int* __restrict__ fo, const int* __restrict__ wscan,
                             const int* __restrict__ pscan, int P, int* __restrict__ counts,
                             int* __restrict__ so, PadCaps pc, int* __restrict__ status) {
  HF_PDL_ENTRY();
  __shared__ int ns[HF_MAX_T];
  const int t = threadIdx.x;
  if (t < m.T) {
    const int nd = fo[t + 1] - fo[t];
    const int nn = wscan[m.wbase[t + 1]] - wscan[m.wbase[t]];
    ns[t] = nd + nn;
    counts[t] = nd + nn;
    counts[m.T + t] = nd;
    if (pc.on && nd + nn > pc.off[t + 1] - pc.off[t]) atomicOr(status, HIFUSE_ST_OVERFLOW);
  }
  __syncthreads();
  if (t == 0) {
    int a = 0;
    for (int q = 0; q < m.T; q++) {
      so[q] = pc.on ? pc.off[q] : a;
      a += ns[q];
    }
    so[m.T] = pc.on ? pc.off[m.T] : a;
    counts[2 * m.T] = pscan[P];
    if (pc.on && pscan[P] > pc.ecap) atomicOr(status, HIFUSE_ST_OVERFLOW);
  }
}

__global__ void __launch_bounds__(256)
k_smp_assign(SmpMeta m, int W, const int* __restrict__ fo_d, const int* __restrict__ so_d,
             const int* __restrict__ front, const unsigned* __restrict__ bitmap,
             const int* __restrict__ wscan, int* __restrict__ loc, int* __restrict__ src_gid) {
  HF_PDL_ENTRY();
  __shared__ int fo[HF_MAX_T + 1], so[HF_MAX_T + 1];
  for (int i = threadIdx.x; i <= m.T; i += blockDim.x) { fo[i] = fo_d[i]; so[i] = so_d[i]; }
  __syncthreads();
  const long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (x < W) {                                   // new sources: n_dst + rank
    const int w = (int)x;
    unsigned bits = bitmap[w];
    if (!bits) return;
    int s = 0;
    while (s + 1 < m.T && m.wbase[s + 1] <= w) s++;
    const int nd = fo[s + 1] - fo[s];
    const int r0 = wscan[w] - wscan[m.wbase[s]];
    int k = 0;
    const int cap = so[s + 1] - so[s];            // (padded layout: overflow past it)
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int u = (w - m.wbase[s]) * 32 + b;
      const int l = nd + r0 + k++;
      loc[m.goff[s] + u] = l;
      if (l < cap) src_gid[so[s] + l] = u;
    }
  } else {                                       // destinations: the prefix
    const long long d = x - W;
    if (d >= fo[m.T]) return;
    const int t = type_of(fo, m.T, (int)d);
    src_gid[so[t] + (d - fo[t])] = front[d];
  }
}

// Compaction of the slots into (src_local, dst_local, eid): thread per
// (pair, pick) slot.  Padded layout: positions [N, ecap) become null edges.
__global__ void __launch_bounds__(256)
k_smp_edges(SmpMeta m, int f, long long nslots, const int* __restrict__ fo_d,
            const int* __restrict__ pair_cnt, const int* __restrict__ pscan, int P,
            const int* __restrict__ slot_src, const long long* __restrict__ slot_eid,
            const int* __restrict__ loc, int* __restrict__ src_local,
            int* __restrict__ dst_local, long long* __restrict__ edge_id, long long ecap,
            const int* __restrict__ so_d) {
  HF_PDL_ENTRY();
  __shared__ int fo[HF_MAX_T + 1], so[HF_MAX_T + 1];
  for (int i = threadIdx.x; i <= m.T; i += blockDim.x) { fo[i] = fo_d[i]; so[i] = so_d[i]; }
  __syncthreads();
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long x0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (ecap >= 0)                                  // padded layout: null edges at [N, ecap)
    for (long long x = pscan[P] + x0; x < ecap; x += nth) {
      src_local[x] = 0;
      dst_local[x] = 0;
      edge_id[x] = -1;
    }
  // slots of the actual frontier's pairs (pair_cnt past it was never written)
  const long long nact = min(nslots, (long long)fo[m.T] * m.Rmax * f);
  for (long long x = x0; x < nact; x += nth) {
  const int p = (int)(x / f), j = (int)(x % f);
  if (j >= pair_cnt[p]) continue;
  const int pos = pscan[p] + j;
  if (ecap >= 0 && pos >= ecap) continue;         // overflow (flagged by k_smp_counts)
  const int d = p / m.Rmax, q = p % m.Rmax;
  const int t = type_of(fo, m.T, d);
  const int r = m.trel[m.trel_off[t] + q];
  const int s = m.rel_src[r];
  const int ls = loc[m.goff[s] + slot_src[x]];
  if (ecap >= 0 && ls >= so[s + 1] - so[s]) {     // overflowed source: null edge (the block
    src_local[pos] = 0;                           // stays a valid, truncated one; the caller
    dst_local[pos] = 0;                           // re-samples it, HIFUSE_ST_OVERFLOW)
    edge_id[pos] = -1;
    continue;
  }
  src_local[pos] = ls;
  dst_local[pos] = d - fo[t];
  edge_id[pos] = slot_eid[x];
  }
}

__global__ void __launch_bounds__(256)
k_smp_gather(SmpMeta m, const int* __restrict__ so_d, const int* __restrict__ src_gid,
             int* __restrict__ gather_ids) {
  HF_PDL_ENTRY();
  __shared__ int so[HF_MAX_T + 1];
  for (int i = threadIdx.x; i <= m.T; i += blockDim.x) so[i] = so_d[i];
  __syncthreads();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < so[m.T]; x += gridDim.x * blockDim.x) {
    const int t = type_of(so, m.T, x);
    gather_ids[x] = (int)(m.goff[t] + max(src_gid[x], 0));   // padding slot: the type's row 0
  }
}

struct SmpPlan {
  int L, T, R, Rmax, W;
  long long Vtot;
  std::vector<long long> D, P, E, S;     // per hop (innermost layer first)
  long long Pmax, Smax, Dmax;
};

static hifuse_status make_plan(const hifuse_graph_csc* g, int L, const int32_t* fan,
                               int64_t B, SmpPlan* pl) {
  if (!g || !fan || L < 1 || B < 0 || g->num_types < 1 || g->num_types > HF_MAX_T ||
      g->num_rels < 0 || g->num_rels > HF_MAX_R || !g->type_count_h || !g->in_ptr_off_h ||
      (g->num_rels > 0 && (!g->rel_src_type_h || !g->rel_dst_type_h)))
    return HIFUSE_ERR_INVALID_ARG;
  pl->L = L;
  pl->T = g->num_types;
  pl->R = g->num_rels;
  pl->Vtot = 0;
  pl->W = 0;
  for (int t = 0; t < pl->T; t++) {
    if (g->type_count_h[t] < 0) return HIFUSE_ERR_INVALID_ARG;
    pl->Vtot += g->type_count_h[t];
    pl->W += (int)((g->type_count_h[t] + 31) / 32);
  }
  if (pl->Vtot >= (1ll << 31)) return HIFUSE_ERR_UNSUPPORTED;
  int rmax = 0;
  for (int t = 0; t < pl->T; t++) {
    int c = 0;
    for (int r = 0; r < pl->R; r++) {
      if (g->rel_src_type_h[r] < 0 || g->rel_src_type_h[r] >= pl->T || g->rel_dst_type_h[r] < 0 ||
          g->rel_dst_type_h[r] >= pl->T)
        return HIFUSE_ERR_INVALID_ARG;
      c += g->rel_dst_type_h[r] == t;
    }
    rmax = std::max(rmax, c);
  }
  pl->Rmax = std::max(rmax, 1);
  pl->D.assign(L, 0); pl->P.assign(L, 0); pl->E.assign(L, 0); pl->S.assign(L, 0);
  long long D = B;
  pl->Pmax = pl->Smax = pl->Dmax = 1;
  for (int h = 0; h < L; h++) {
    const int f = fan[L - 1 - h];
    if (f < 1 || f > kMaxFan) return HIFUSE_ERR_INVALID_ARG;
    pl->D[h] = D;
    pl->P[h] = D * pl->Rmax;
    pl->E[h] = pl->P[h] * f;
    pl->S[h] = std::min(D + pl->E[h], pl->Vtot);
    if (pl->E[h] >= (1ll << 31)) return HIFUSE_ERR_UNSUPPORTED;
    pl->Pmax = std::max(pl->Pmax, pl->P[h]);
    pl->Smax = std::max(pl->Smax, pl->E[h]);
    pl->Dmax = std::max(pl->Dmax, D);
    D = pl->S[h];
  }
  return HIFUSE_OK;
}

static size_t plan_ws(const SmpPlan& pl) {
  return carve_bytes(pl.Smax, 4) + carve_bytes(pl.Smax, 8) + carve_bytes(pl.Pmax, 4) +
         carve_bytes(pl.Pmax + 1, 4) + carve_bytes(scan_ws_ints(pl.Pmax), 4) +
         carve_bytes(std::max(pl.W, 1), 4) * 2 + carve_bytes(pl.W + 1, 4) +
         carve_bytes(scan_ws_ints(std::max(pl.W, 1)), 4) + 2 * carve_bytes(HF_MAX_T + 1, 4);
}

}  // namespace hf

using namespace hf;

extern "C" {

hifuse_status hifuse_sample_caps(const hifuse_graph_csc* g, int num_layers, const int32_t* fanout_h,
                                 int64_t num_seeds, int64_t* edge_cap_h, int64_t* src_cap_h,
                                 size_t* ws_bytes, int64_t* state_ints) {
  SmpPlan pl;
  hifuse_status rc = make_plan(g, num_layers, fanout_h, num_seeds, &pl);
  if (rc != HIFUSE_OK) return rc;
  for (int h = 0; h < num_layers; h++) {
    const int l = num_layers - 1 - h;
    if (edge_cap_h) edge_cap_h[l] = std::max(pl.E[h], 1ll);
    if (src_cap_h) src_cap_h[l] = std::max(pl.S[h], 1ll);
  }
  if (ws_bytes) *ws_bytes = plan_ws(pl);
  if (state_ints) *state_ints = 2 * std::max(pl.Vtot, 1ll);
  return HIFUSE_OK;
}

}  // extern "C"

// Shared body of hifuse_sample_blocks (compact layout: src_cap_h == NULL) and
// hifuse_sample_blocks_padded (per-type source capacities, padded edge tail).
static hifuse_status sample_impl(const hifuse_graph_csc* g, int num_layers,
                                 const int32_t* fanout_h, const int32_t* d_seeds,
                                 int64_t num_seeds, int32_t target_type, uint64_t key,
                                 const uint64_t* d_ctl, int32_t stamp, const int64_t* src_cap_h,
                                 const int64_t* edge_pad_h, hifuse_block* out, int32_t* d_state,
                                 void* d_ws, size_t ws_bytes, int32_t* d_status,
                                 hifuse_stream_t stream) {
  SmpPlan pl;
  hifuse_status rc = make_plan(g, num_layers, fanout_h, num_seeds, &pl);
  if (rc != HIFUSE_OK) return rc;
  const bool padded = src_cap_h != nullptr;
  if (padded) {
    // per layer l: caps >= 0, sum <= the worst-case source capacity; the
    // layer's destinations (layer l+1's sources, or the seeds) fit its sources;
    // the padded edge count <= the worst-case edge capacity
    if (!edge_pad_h) return HIFUSE_ERR_INVALID_ARG;
    for (int h = 0; h < num_layers; h++) {
      const int l = num_layers - 1 - h;
      long long tot = 0;
      for (int t = 0; t < pl.T; t++) {
        const long long c = src_cap_h[(long long)l * pl.T + t];
        const long long d = l == num_layers - 1 ? (t == target_type ? num_seeds : 0)
                                                : src_cap_h[(long long)(l + 1) * pl.T + t];
        if (c < 0 || c < d) return HIFUSE_ERR_INVALID_ARG;
        tot += c;
      }
      if (tot > pl.S[h] || edge_pad_h[l] < 0 || edge_pad_h[l] > pl.E[h])
        return HIFUSE_ERR_INVALID_ARG;
    }
  }
  if (target_type < 0 || target_type >= pl.T || stamp < 1 || !d_state || !d_status || !out ||
      (num_seeds > 0 && !d_seeds) || !g->d_in_ptr || (pl.R > 0 && (!g->d_in_src || !g->d_in_eid)))
    return HIFUSE_ERR_INVALID_ARG;
  for (int l = 0; l < num_layers; l++)
    if (!out[l].src_local || !out[l].dst_local || !out[l].edge_id || !out[l].src_gid ||
        !out[l].counts)
      return HIFUSE_ERR_INVALID_ARG;
  if (ws_bytes < plan_ws(pl) || !d_ws) return HIFUSE_ERR_WORKSPACE;
  SmpMeta m;
  m.T = pl.T;
  m.R = pl.R;
  m.Rmax = pl.Rmax;
  m.goff[0] = 0;
  m.wbase[0] = 0;
  for (int t = 0; t < pl.T; t++) {
    m.count[t] = g->type_count_h[t];
    m.goff[t + 1] = m.goff[t] + g->type_count_h[t];
    m.wbase[t + 1] = m.wbase[t] + (int)((g->type_count_h[t] + 31) / 32);
  }
  int q = 0;
  for (int t = 0; t < pl.T; t++) {
    m.trel_off[t] = q;
    for (int r = 0; r < pl.R; r++)
      if (g->rel_dst_type_h[r] == t) m.trel[q++] = r;
  }
  m.trel_off[pl.T] = q;
  for (int r = 0; r < pl.R; r++) {
    m.rel_src[r] = g->rel_src_type_h[r];
    m.in_ptr_off[r] = g->in_ptr_off_h[r];
  }
  cudaStream_t s = st(stream);
  char* p = (char*)d_ws;
  int* slot_src = carve<int>(p, pl.Smax);
  long long* slot_eid = carve<long long>(p, pl.Smax);
  int* pair_cnt = carve<int>(p, pl.Pmax);
  int* pscan = carve<int>(p, pl.Pmax + 1);
  int* pscan_ws = carve<int>(p, scan_ws_ints(pl.Pmax));
  unsigned* bitmap = carve<unsigned>(p, std::max(pl.W, 1));
  int* wcnt = carve<int>(p, std::max(pl.W, 1));
  int* wscan = carve<int>(p, pl.W + 1);
  int* wscan_ws = carve<int>(p, scan_ws_ints(std::max(pl.W, 1)));
  int* fo_a = carve<int>(p, HF_MAX_T + 1);
  int* fo_b = carve<int>(p, HF_MAX_T + 1);
  int* gen = d_state;
  int* loc = d_state + pl.Vtot;
  HF_LAUNCH(k_smp_init, 1, HF_MAX_T + 1, 0, s, pl.T, target_type, (int)num_seeds, fo_a);
  const int* front = d_seeds;
  int* fo = fo_a;
  int* so = fo_b;
  for (int h = 0; h < num_layers; h++) {
    const int l = num_layers - 1 - h;
    const int f = fanout_h[l];
    const unsigned long long hk = [&] {
      unsigned long long z = key ^ (0x1000ull + (unsigned long long)h);
      z += 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    }();
    const int stp = stamp + h;
    hifuse_block& o = out[l];
    const long long D = pl.D[h], P = pl.P[h];
    PadCaps pc;
    memset(&pc, 0, sizeof(pc));
    pc.ecap = -1;
    long long cap_tot = 0;
    if (padded) {
      pc.on = 1;
      for (int t = 0; t < pl.T; t++) {
        pc.off[t] = (int)cap_tot;
        cap_tot += src_cap_h[(long long)l * pl.T + t];
      }
      pc.off[pl.T] = (int)cap_tot;
      pc.ecap = edge_pad_h[l];
      // padding slots of the type-major source list read -1
      cudaMemsetAsync(o.src_gid, 0xff, sizeof(int) * std::max(cap_tot, 1ll), s);
    }
    cudaMemsetAsync(bitmap, 0, sizeof(unsigned) * std::max(pl.W, 1), s);
    HF_LAUNCH(k_smp_mark_dst, ceil_div(D, 256), 256, 0, s, m, fo, front, gen, loc, stp,
              (const unsigned long long*)d_ctl, h, padded && h > 0 ? 1 : 0, d_status);
    // Grid-stride kernels, sized to the frontier's bound: the padded layout
    // knows it on the host (the seeds, or the previous hop's capacities), so
    // every warp gets one pair and then exits -- a persistent grid held every
    // SM's warp slots for the whole pair kernel and starved the training step
    // it runs beside (SampledLoop); the compact layout only knows the
    // worst case and keeps one resident wave.
    long long front_cap = D;
    if (padded && h > 0) {
      front_cap = 0;
      for (int t = 0; t < pl.T; t++) front_cap += src_cap_h[(long long)(l + 1) * pl.T + t];
    }
    const long long pair_bound = std::min<long long>(P, front_cap * pl.Rmax);
    const long long cap_blocks = (long long)sm_count() * 8;
    auto gs_grid = [&](long long work, long long per_block) -> long long {
      const long long g = std::max<long long>(1, (long long)ceil_div(work, per_block));
      return padded ? g : std::min(g, cap_blocks);
    };
    HF_LAUNCH(k_smp_pairs, gs_grid(pair_bound, kSmpWarps), kSmpWarps * 32, 0, s, m, fo, front, (int)P, f, hk,
              (const unsigned long long*)d_ctl, h, (const long long*)g->d_in_ptr, g->d_in_src, (const long long*)g->d_in_eid, gen,
              bitmap, stp, slot_src, slot_eid, pair_cnt);
    HF_LAUNCH(k_smp_popc, ceil_div(pl.W, 256), 256, 0, s, bitmap, pl.W, wcnt);
    exclusive_scan(wcnt, wscan, pl.W, wscan_ws, s);
    exclusive_scan(pair_cnt, pscan, P, pscan_ws, s);
    HF_LAUNCH(k_smp_counts, 1, HF_MAX_T, 0, s, m, fo, wscan, pscan, (int)P, o.counts, so, pc,
              d_status);
    HF_LAUNCH(k_smp_assign, ceil_div(pl.W + D, 256), 256, 0, s, m, pl.W, fo, so, front, bitmap,
              wscan, loc, o.src_gid);
    HF_LAUNCH(k_smp_edges, gs_grid(pair_bound * f, 256 * 4), 256, 0, s, m, f, P * f, fo, pair_cnt, pscan,
              (int)P, slot_src, slot_eid, loc, o.src_local, o.dst_local, (long long*)o.edge_id,
              pc.ecap, so);
    if (o.gather_ids)
      HF_LAUNCH(k_smp_gather, gs_grid(padded ? std::max(cap_tot, 1ll) : pl.S[h], 256 * 4), 256, 0,
                s, m, so, o.src_gid, o.gather_ids);
    front = o.src_gid;
    std::swap(fo, so);
  }
  return last_cuda();
}

extern "C" {

hifuse_status hifuse_sample_blocks(const hifuse_graph_csc* g, int num_layers,
                                   const int32_t* fanout_h, const int32_t* d_seeds,
                                   int64_t num_seeds, int32_t target_type, uint64_t key,
                                   const uint64_t* d_ctl, int32_t stamp, hifuse_block* out,
                                   int32_t* d_state,
                                   void* d_ws, size_t ws_bytes, int32_t* d_status,
                                   hifuse_stream_t stream) {
  return sample_impl(g, num_layers, fanout_h, d_seeds, num_seeds, target_type, key, d_ctl, stamp,
                     nullptr, nullptr, out, d_state, d_ws, ws_bytes, d_status, stream);
}

hifuse_status hifuse_sample_blocks_padded(const hifuse_graph_csc* g, int num_layers,
                                          const int32_t* fanout_h, const int32_t* d_seeds,
                                          int64_t num_seeds, int32_t target_type, uint64_t key,
                                          const uint64_t* d_ctl, int32_t stamp,
                                          const int64_t* src_cap_h, const int64_t* edge_pad_h,
                                          hifuse_block* out, int32_t* d_state, void* d_ws,
                                          size_t ws_bytes, int32_t* d_status,
                                          hifuse_stream_t stream) {
  if (!src_cap_h || !edge_pad_h) return HIFUSE_ERR_INVALID_ARG;
  return sample_impl(g, num_layers, fanout_h, d_seeds, num_seeds, target_type, key, d_ctl, stamp,
                     src_cap_h, edge_pad_h, out, d_state, d_ws, ws_bytes, d_status, stream);
}
}  // extern "C"

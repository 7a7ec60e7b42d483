// sample.cu -- GPU neighbour sampler (Fig. 2
// step (1), line 156; SPEC.md sample_batch S:L126-143).  include/hifuse.h
// documents the contract.  Per hop (innermost layer first), 7 kernels and two
// scans, independent of R and of the batch:
//   k_smp_mark_dst  destinations: gen[v] = stamp, loc[v] = local id
//   k_smp_pairs     thread per (destination, relation into its type): Floyd's
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
#include <vector>
#include "common.cuh"

namespace hf {

static constexpr int kMaxFan = 64;

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
  int t = threadIdx.x;
  if (t <= T) fo[t] = t <= target ? 0 : B;
}

__global__ void __launch_bounds__(256)
k_smp_mark_dst(SmpMeta m, const int* __restrict__ fo_d, const int* __restrict__ front,
               int* __restrict__ gen, int* __restrict__ loc, int stamp,
               const unsigned long long* __restrict__ d_ctl, int hop, int* __restrict__ status) {
  __shared__ int fo[HF_MAX_T + 1];
  for (int i = threadIdx.x; i <= m.T; i += blockDim.x) fo[i] = fo_d[i];
  __syncthreads();
  if (d_ctl) stamp = (int)d_ctl[1] + hop;
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= fo[m.T]) return;
  const int t = type_of(fo, m.T, d);
  const int v = front[d];
  if (v < 0 || v >= m.count[t]) {
    atomicOr(status, HIFUSE_ST_BAD_DST);
    return;
  }
  const long long g = m.goff[t] + v;
  gen[g] = stamp;
  loc[g] = d - fo[t];
}

__global__ void __launch_bounds__(128)
k_smp_pairs(SmpMeta m, const int* __restrict__ fo_d, const int* __restrict__ front, int P, int f,
            unsigned long long hk, const unsigned long long* __restrict__ d_ctl, int hop,
            const long long* __restrict__ in_ptr,
            const int* __restrict__ in_src, const long long* __restrict__ in_eid,
            int* __restrict__ gen, unsigned* __restrict__ bitmap, int stamp,
            int* __restrict__ slot_src, long long* __restrict__ slot_eid,
            int* __restrict__ pair_cnt) {
  __shared__ int fo[HF_MAX_T + 1];
  for (int i = threadIdx.x; i <= m.T; i += blockDim.x) fo[i] = fo_d[i];
  __syncthreads();
  if (d_ctl) {                       // key and stamp base from device memory
    hk = mix64(d_ctl[0] ^ (0x1000ull + (unsigned long long)hop));
    stamp = (int)d_ctl[1] + hop;
  }
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int d = p / m.Rmax, q = p % m.Rmax;
  int k = 0;
  if (d < fo[m.T]) {
    const int t = type_of(fo, m.T, d);
    const int v = front[d];
    if (q < m.trel_off[t + 1] - m.trel_off[t] && v >= 0 && v < m.count[t]) {
      const int r = m.trel[m.trel_off[t] + q];
      const long long* ptr = in_ptr + m.in_ptr_off[r] + v;
      const long long base = ptr[0];
      const int deg = (int)(ptr[1] - base);
      k = min(deg, f);
      int sel[kMaxFan];
      if (deg <= f) {
        for (int j = 0; j < k; j++) sel[j] = j;
      } else {
        // Floyd: for j = deg-k .. deg-1, t = U[0, j]; take t unless taken, else j
        int n = 0;
        for (int j = deg - k; j < deg; j++) {
          const int c = rand_upto(hk, r, v, j);
          bool taken = false;
          for (int a = 0; a < n; a++) taken |= sel[a] == c;
          sel[n++] = taken ? j : c;
        }
        for (int a = 1; a < k; a++) {                 // ascending in-list order
          const int x = sel[a];
          int b = a - 1;
          while (b >= 0 && sel[b] > x) { sel[b + 1] = sel[b]; b--; }
          sel[b + 1] = x;
        }
      }
      const int s = m.rel_src[r];
      for (int j = 0; j < k; j++) {
        const long long e = base + sel[j];
        const int u = in_src[e];
        if (atomicExch(gen + m.goff[s] + u, stamp) != stamp)
          atomicOr(bitmap + m.wbase[s] + (u >> 5), 1u << (u & 31));
        slot_src[(long long)p * f + j] = u;
        slot_eid[(long long)p * f + j] = in_eid[e];
      }
    }
  }
  pair_cnt[p] = k;
}

__global__ void k_smp_popc(const unsigned* __restrict__ bitmap, int W, int* __restrict__ wcnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < W) wcnt[i] = __popc(bitmap[i]);
}

__global__ void k_smp_counts(SmpMeta m, const int* __restrict__ fo, const int* __restrict__ wscan,
                             const int* __restrict__ pscan, int P, int* __restrict__ counts,
                             int* __restrict__ so) {
  __shared__ int ns[HF_MAX_T];
  const int t = threadIdx.x;
  if (t < m.T) {
    const int nd = fo[t + 1] - fo[t];
    const int nn = wscan[m.wbase[t + 1]] - wscan[m.wbase[t]];
    ns[t] = nd + nn;
    counts[t] = nd + nn;
    counts[m.T + t] = nd;
  }
  __syncthreads();
  if (t == 0) {
    int a = 0;
    for (int q = 0; q < m.T; q++) { so[q] = a; a += ns[q]; }
    so[m.T] = a;
    counts[2 * m.T] = pscan[P];
  }
}

__global__ void __launch_bounds__(256)
k_smp_assign(SmpMeta m, int W, const int* __restrict__ fo_d, const int* __restrict__ so_d,
             const int* __restrict__ front, const unsigned* __restrict__ bitmap,
             const int* __restrict__ wscan, int* __restrict__ loc, int* __restrict__ src_gid) {
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
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int u = (w - m.wbase[s]) * 32 + b;
      const int l = nd + r0 + k++;
      loc[m.goff[s] + u] = l;
      src_gid[so[s] + l] = u;
    }
  } else {                                       // destinations: the prefix
    const long long d = x - W;
    if (d >= fo[m.T]) return;
    const int t = type_of(fo, m.T, (int)d);
    src_gid[so[t] + (d - fo[t])] = front[d];
  }
}

__global__ void __launch_bounds__(256)
k_smp_edges(SmpMeta m, int f, long long nslots, const int* __restrict__ fo_d,
            const int* __restrict__ pair_cnt, const int* __restrict__ pscan,
            const int* __restrict__ slot_src, const long long* __restrict__ slot_eid,
            const int* __restrict__ loc, int* __restrict__ src_local,
            int* __restrict__ dst_local, long long* __restrict__ edge_id) {
  __shared__ int fo[HF_MAX_T + 1];
  for (int i = threadIdx.x; i <= m.T; i += blockDim.x) fo[i] = fo_d[i];
  __syncthreads();
  const long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nslots) return;
  const int p = (int)(x / f), j = (int)(x % f);
  if (j >= pair_cnt[p]) return;
  const int pos = pscan[p] + j;
  const int d = p / m.Rmax, q = p % m.Rmax;
  const int t = type_of(fo, m.T, d);
  const int r = m.trel[m.trel_off[t] + q];
  const int s = m.rel_src[r];
  src_local[pos] = loc[m.goff[s] + slot_src[x]];
  dst_local[pos] = d - fo[t];
  edge_id[pos] = slot_eid[x];
}

__global__ void __launch_bounds__(256)
k_smp_gather(SmpMeta m, const int* __restrict__ so_d, const int* __restrict__ src_gid,
             int* __restrict__ gather_ids) {
  __shared__ int so[HF_MAX_T + 1];
  for (int i = threadIdx.x; i <= m.T; i += blockDim.x) so[i] = so_d[i];
  __syncthreads();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= so[m.T]) return;
  const int t = type_of(so, m.T, x);
  gather_ids[x] = (int)(m.goff[t] + src_gid[x]);
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

hifuse_status hifuse_sample_blocks(const hifuse_graph_csc* g, int num_layers,
                                   const int32_t* fanout_h, const int32_t* d_seeds,
                                   int64_t num_seeds, int32_t target_type, uint64_t key,
                                   const uint64_t* d_ctl, int32_t stamp, hifuse_block* out,
                                   int32_t* d_state,
                                   void* d_ws, size_t ws_bytes, int32_t* d_status,
                                   hifuse_stream_t stream) {
  SmpPlan pl;
  hifuse_status rc = make_plan(g, num_layers, fanout_h, num_seeds, &pl);
  if (rc != HIFUSE_OK) return rc;
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
    cudaMemsetAsync(bitmap, 0, sizeof(unsigned) * std::max(pl.W, 1), s);
    HF_LAUNCH(k_smp_mark_dst, ceil_div(D, 256), 256, 0, s, m, fo, front, gen, loc, stp,
              (const unsigned long long*)d_ctl, h, d_status);
    HF_LAUNCH(k_smp_pairs, ceil_div(P, 128), 128, 0, s, m, fo, front, (int)P, f, hk,
              (const unsigned long long*)d_ctl, h, (const long long*)g->d_in_ptr, g->d_in_src, (const long long*)g->d_in_eid, gen,
              bitmap, stp, slot_src, slot_eid, pair_cnt);
    HF_LAUNCH(k_smp_popc, ceil_div(pl.W, 256), 256, 0, s, bitmap, pl.W, wcnt);
    exclusive_scan(wcnt, wscan, pl.W, wscan_ws, s);
    exclusive_scan(pair_cnt, pscan, P, pscan_ws, s);
    HF_LAUNCH(k_smp_counts, 1, HF_MAX_T, 0, s, m, fo, wscan, pscan, (int)P, o.counts, so);
    HF_LAUNCH(k_smp_assign, ceil_div(pl.W + D, 256), 256, 0, s, m, pl.W, fo, so, front, bitmap,
              wscan, loc, o.src_gid);
    HF_LAUNCH(k_smp_edges, ceil_div(P * f, 256), 256, 0, s, m, f, P * f, fo, pair_cnt, pscan,
              slot_src, slot_eid, loc, o.src_local, o.dst_local, (long long*)o.edge_id);
    if (o.gather_ids)
      HF_LAUNCH(k_smp_gather, ceil_div(pl.S[h], 256), 256, 0, s, m, so, o.src_gid, o.gather_ids);
    front = o.src_gid;
    std::swap(fo, so);
  }
  return last_cuda();
}

}  // extern "C"

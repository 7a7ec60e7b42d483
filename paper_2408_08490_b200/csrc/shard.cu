// shard.cu -- NEXT(4): feature-sharded data
// parallelism.  PAPER.md line 219 ("a large heterogeneous graph can be
// partitioned into several subgraphs") and line 404: when the type-major
// feature store does not fit one GPU, rank k keeps the row range
// [bounds[k], bounds[k+1]) and every batch fetches the layer-0 rows it
// collects (A2) from their owners with one all-to-all of row ids and one of
// rows (paper_2408_08490_b200/shard.py drives the exchange).  The kernels
// here are the data movement around the exchange:
//   k_shard_plan   stable counting sort of the batch's row ids by owner rank
//                  (one block: W <= 64 owners, ids in batch order inside an
//                  owner), giving per-owner counts and the send order
//   k_gather_words dst[i] = src[idx[i] - base] for rows of `words` 4-byte
//                  words (ids to send, local rows to return; 16-byte vectors
//                  when rows allow)
//   k_scatter_words dst[idx[i]] = src[i] (received rows back to batch order)
#include "common.cuh"

namespace hf {
namespace {

constexpr int kPlanThreads = 1024;

// One block, one pass per owner k (W is small): every thread counts the ids
// of owner k in its contiguous slice, a block-wide exclusive scan gives the
// slice's offset, and the ids are placed in batch order (stable).
__device__ __forceinline__ int block_excl_scan_1024(int v, int* red, int* total) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) red[w] = inc;
  __syncthreads();
  if (w == 0) {
    int x = red[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    red[lane] = x;
  }
  __syncthreads();
  const int ex = (w ? red[w - 1] : 0) + inc - v;
  *total = red[31];
  __syncthreads();
  return ex;
}

__global__ void __launch_bounds__(kPlanThreads)
k_shard_plan(const int* __restrict__ ids, int n, const long long* __restrict__ bounds, int W,
             int* __restrict__ counts, int* __restrict__ order, int* __restrict__ status) {
  HF_PDL_ENTRY();
  __shared__ long long sb[65];
  __shared__ int red[32];
  const int t = threadIdx.x;
  for (int k = t; k <= W; k += kPlanThreads) sb[k] = bounds[k];
  __syncthreads();
  const int per = (n + kPlanThreads - 1) / kPlanThreads;
  const int a = min(n, t * per), b = min(n, a + per);
  auto owner = [&](long long id) {
    if (id < sb[0] || id >= sb[W]) return -1;
    int lo = 0, hi = W;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (sb[mid] <= id) lo = mid; else hi = mid;
    }
    return lo;
  };
  int base = 0;
  for (int k = 0; k < W; k++) {
    int c = 0;
    for (int i = a; i < b; i++) c += owner(ids[i]) == k;
    int total;
    int off = base + block_excl_scan_1024(c, red, &total);
    for (int i = a; i < b; i++)
      if (owner(ids[i]) == k) order[off++] = i;
    if (t == 0) counts[k] = total;
    base += total;
  }
  if (t == 0 && base != n) atomicOr(status, HIFUSE_ST_BAD_EDGE_ID);   // ids outside every shard
}

template <typename V>
__global__ void k_gather_words(const V* __restrict__ src, const int* __restrict__ idx, long long n,
                               int vpr, long long base, V* __restrict__ dst) {
  HF_PDL_ENTRY();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * vpr) return;
  const long long r = i / vpr, c = i % vpr;
  dst[i] = src[(idx[r] - base) * vpr + c];
}

template <typename V>
__global__ void k_scatter_words(const V* __restrict__ src, const int* __restrict__ idx,
                                long long n, int vpr, V* __restrict__ dst) {
  HF_PDL_ENTRY();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * vpr) return;
  const long long r = i / vpr, c = i % vpr;
  dst[(long long)idx[r] * vpr + c] = src[i];
}

}  // namespace
}  // namespace hf

using namespace hf;

extern "C" {

hifuse_status hifuse_shard_plan(const int32_t* d_ids, int64_t n, const int64_t* d_bounds, int W,
                                int32_t* d_counts, int32_t* d_order, int32_t* d_status,
                                hifuse_stream_t stream) {
  if (n < 0 || n >= (1ll << 31) || W <= 0 || W > 64 || !d_bounds || !d_counts || !d_status ||
      (n > 0 && (!d_ids || !d_order)))
    return HIFUSE_ERR_INVALID_ARG;
  HF_LAUNCH(k_shard_plan, 1, kPlanThreads, 0, st(stream), d_ids, (int)n,
            (const long long*)d_bounds, W, d_counts, d_order, d_status);
  return last_cuda();
}

hifuse_status hifuse_gather_words(const void* d_src, const int32_t* d_idx, int64_t n, int words,
                                  int64_t base, void* d_dst, hifuse_stream_t stream) {
  if (n < 0 || words <= 0 || (n > 0 && (!d_src || !d_idx || !d_dst))) return HIFUSE_ERR_INVALID_ARG;
  if (n == 0) return HIFUSE_OK;
  cudaStream_t s = st(stream);
  if (words % 4 == 0 && aligned16(d_src) && aligned16(d_dst)) {
    const long long tot = n * (words / 4);
    HF_LAUNCH(k_gather_words<int4>, ceil_div(tot, 256), 256, 0, s, (const int4*)d_src, d_idx,
              (long long)n, words / 4, (long long)base, (int4*)d_dst);
  } else {
    const long long tot = n * words;
    HF_LAUNCH(k_gather_words<int>, ceil_div(tot, 256), 256, 0, s, (const int*)d_src, d_idx,
              (long long)n, words, (long long)base, (int*)d_dst);
  }
  return last_cuda();
}

hifuse_status hifuse_scatter_words(const void* d_src, const int32_t* d_idx, int64_t n, int words,
                                   void* d_dst, hifuse_stream_t stream) {
  if (n < 0 || words <= 0 || (n > 0 && (!d_src || !d_idx || !d_dst))) return HIFUSE_ERR_INVALID_ARG;
  if (n == 0) return HIFUSE_OK;
  cudaStream_t s = st(stream);
  if (words % 4 == 0 && aligned16(d_src) && aligned16(d_dst)) {
    const long long tot = n * (words / 4);
    HF_LAUNCH(k_scatter_words<int4>, ceil_div(tot, 256), 256, 0, s, (const int4*)d_src, d_idx,
              (long long)n, words / 4, (int4*)d_dst);
  } else {
    const long long tot = n * words;
    HF_LAUNCH(k_scatter_words<int>, ceil_div(tot, 256), 256, 0, s, (const int*)d_src, d_idx,
              (long long)n, words, (int*)d_dst);
  }
  return last_cuda();
}

}  // extern "C"

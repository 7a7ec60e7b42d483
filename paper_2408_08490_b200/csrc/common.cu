// common.cu -- layer metadata, device-wide scan, status helpers.
#include "common.cuh"

#include <map>
#include <mutex>
#include <set>

namespace hf {

std::atomic<int64_t> g_launches{0};

hifuse_status make_meta(const hifuse_layer_shape* s, LayerMeta* m) {
  if (!s || !m) return HIFUSE_ERR_INVALID_ARG;
  if (s->num_types <= 0 || s->num_types > HF_MAX_T) return HIFUSE_ERR_UNSUPPORTED;
  if (s->num_rels <= 0 || s->num_rels > HF_MAX_R) return HIFUSE_ERR_UNSUPPORTED;
  if (!s->rel_src_type_h || !s->rel_dst_type_h || !s->n_src_h || !s->n_dst_h)
    return HIFUSE_ERR_INVALID_ARG;
  if (s->num_edges < 0 || s->num_edges >= (1ll << 31)) return HIFUSE_ERR_INVALID_ARG;
  m->T = s->num_types;
  m->R = s->num_rels;
  m->N = (int)s->num_edges;
  long long so = 0, dof = 0;
  for (int t = 0; t < m->T; t++) {
    int ns = s->n_src_h[t], nd = s->n_dst_h[t];
    if (ns < 0 || nd < 0 || nd > ns) return HIFUSE_ERR_INVALID_ARG;
    m->n_src[t] = ns;
    m->n_dst[t] = nd;
    m->type_src_off[t] = (int)so;
    m->type_dst_off[t] = (int)dof;
    so += ns;
    dof += nd;
  }
  m->type_src_off[m->T] = (int)so;
  m->type_dst_off[m->T] = (int)dof;
  long long rows = 0, S = 0;
  for (int r = 0; r < m->R; r++) {
    int a = s->rel_src_type_h[r], b = s->rel_dst_type_h[r];
    if (a < 0 || a >= m->T || b < 0 || b >= m->T) return HIFUSE_ERR_INVALID_ARG;
    m->rel_src[r] = a;
    m->rel_dst[r] = b;
    m->rel_row_off[r] = (int)rows;
    m->slot_off[r] = (int)S;
    rows += m->n_dst[b];
    S += m->n_src[a];
  }
  m->rel_row_off[m->R] = (int)rows;
  m->slot_off[m->R] = (int)S;
  if (so >= (1ll << 31) || rows >= (1ll << 31) || S >= (1ll << 31)) return HIFUSE_ERR_UNSUPPORTED;
  m->rows = (int)rows;
  m->S = (int)S;
  m->src_rows = (int)so;
  m->dst_rows = (int)dof;
  return HIFUSE_OK;
}

// ------------------------------------------------------- per-stream state ---
// Fork/join resources (auxiliary streams + events) are owned per (device,
// caller stream): calls issued on different streams (or from different host
// threads, one stream each) never share an event or a side stream, so there
// is no hidden cross-stream dependency and no record/wait race.  The map is
// mutex-protected; entries are created on first use or by
// hifuse_stream_attach (outside graph capture), and freed by
// hifuse_stream_release.
namespace {
struct StreamKey {
  int dev;
  cudaStream_t s;
  bool operator<(const StreamKey& o) const { return dev != o.dev ? dev < o.dev : s < o.s; }
};
std::mutex g_mu;
std::map<StreamKey, StreamCtx*> g_ctx;
std::map<std::pair<int, const void*>, int> g_smem;
int g_sm[64] = {};
}  // namespace

static StreamCtx* make_ctx() {
  StreamCtx* c = new StreamCtx();
  for (int i = 0; i < kBranches; i++) {
    Branch& n = c->br[i];
    if (cudaStreamCreateWithFlags(&n.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&n.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&n.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      c->ok = false;
      return c;
    }
  }
  if (cudaEventCreateWithFlags(&c->fold, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    c->ok = false;
    return c;
  }
  c->ok = true;
  return c;
}

StreamCtx* stream_ctx(cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_ctx.find(StreamKey{dev, s});
  if (it != g_ctx.end()) return it->second->ok ? it->second : nullptr;
  StreamCtx* c = make_ctx();
  g_ctx[StreamKey{dev, s}] = c;
  return c->ok ? c : nullptr;
}

bool branch_begin(cudaStream_t main, Branch* b, int idx) {
  if (idx < 0 || idx >= kBranches) return false;
  StreamCtx* c = stream_ctx(main);
  if (!c) return false;                  // run the branch serially on `main`
  *b = c->br[idx];
  cudaEventRecord(b->fork, main);
  cudaStreamWaitEvent(b->side, b->fork, 0);
  return true;
}

void branch_end(cudaStream_t main, const Branch& b) {
  cudaEventRecord(b.join, b.side);
  cudaStreamWaitEvent(main, b.join, 0);
}

void set_max_smem(const void* kernel, int bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lk(g_mu);
  int& cur = g_smem[{dev, kernel}];
  if (bytes <= cur) return;
  // raised to the largest request seen so far on this device
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) ==
      cudaSuccess)
    cur = bytes;
  else
    cudaGetLastError();
}

int sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = __atomic_load_n(&g_sm[dev], __ATOMIC_RELAXED);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
    v = 148;
  __atomic_store_n(&g_sm[dev], v, __ATOMIC_RELAXED);
  return v;
}

// ------------------------------------------------------------------ scan ---
static constexpr int kScanThreads = 256;
static constexpr int kScanItems = 32;
static constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ int block_excl_scan(int v, int* total) {
  __shared__ int warp_sums[kScanThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = warp_incl_scan(v);
  if (lane == 31) warp_sums[w] = inc;
  __syncthreads();
  if (w == 0) {
    int s = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
    s = warp_incl_scan(s);
    if (lane < kScanThreads / 32) warp_sums[lane] = s;
  }
  __syncthreads();
  int base = w ? warp_sums[w - 1] : 0;
  *total = warp_sums[kScanThreads / 32 - 1];
  __syncthreads();
  return base + inc - v;
}

// Single-pass exclusive scan with decoupled look-back (tiles claimed in
// order through an atomic ticket, so every predecessor is already running).
// status[t] = (flag << 30) | value: flag 1 = tile aggregate, 2 = inclusive
// prefix.  Values must stay below 2^30 (counts of edges / rows / slots).
// Tile I/O goes through shared memory: coalesced global loads/stores
// (striped over the block), while each thread scans kScanItems consecutive
// items read from a padded layout (index i stored at i + i/32: the 32 items
// of a thread sit in 32 distinct banks).
__device__ __forceinline__ int pad32(int i) { return i + (i >> 5); }

__global__ void __launch_bounds__(kScanThreads)
k_scan_lookback(const int* __restrict__ in, long long n, int* __restrict__ out,
                int* __restrict__ ticket, int* __restrict__ status) {
  HF_PDL_ENTRY();
  __shared__ int s_tile, s_prefix;
  __shared__ int sm[kScanTile + kScanTile / 32];
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int tile = s_tile;
  const long long t0 = (long long)tile * kScanTile;
  const int nt = (int)(n - t0 < kScanTile ? n - t0 : kScanTile);
#pragma unroll
  for (int j = 0; j < kScanItems; j++) {           // coalesced, all loads in flight
    const int i = j * kScanThreads + threadIdx.x;
    sm[pad32(i)] = i < nt ? in[t0 + i] : 0;
  }
  __syncthreads();
  int v[kScanItems];
  int sum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; j++) {
    v[j] = sm[pad32(threadIdx.x * kScanItems + j)];
    sum += v[j];
  }
  int tot;
  int ex = block_excl_scan(sum, &tot);
  if (threadIdx.x < 32) {
    // warp-parallel look-back over a window of 32 predecessors
    volatile int* st_ = status;
    const int lane = threadIdx.x;
    if (tile == 0) {
      if (lane == 0) st_[0] = (2 << 30) | tot;
      if (lane == 0) s_prefix = 0;
    } else {
      if (lane == 0) st_[tile] = (1 << 30) | tot;
      __threadfence();
      int prefix = 0;
      int hi = tile - 1;                       // highest predecessor not yet summed
      while (true) {
        const int t = hi - lane;
        int w = t >= 0 ? st_[t] : (2 << 30);
        int flag = (w >> 30) & 3;
        if (__any_sync(0xffffffffu, flag == 0)) continue;     // someone not published yet
        const unsigned incl = __ballot_sync(0xffffffffu, flag == 2);
        const int stop = incl ? __ffs(incl) - 1 : 32;          // nearest inclusive prefix
        int v2 = (lane <= stop && t >= 0) ? (w & 0x3fffffff) : 0;
        for (int o = 16; o; o >>= 1) v2 += __shfl_xor_sync(0xffffffffu, v2, o);
        prefix += v2;
        if (incl) break;
        hi -= 32;
      }
      if (lane == 0) {
        st_[tile] = (2 << 30) | (prefix + tot);
        s_prefix = prefix;
      }
    }
  }
  __syncthreads();
  ex += s_prefix;
#pragma unroll
  for (int j = 0; j < kScanItems; j++) {
    sm[pad32(threadIdx.x * kScanItems + j)] = ex;
    ex += v[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kScanItems; j++) {           // coalesced stores
    const int i = j * kScanThreads + threadIdx.x;
    if (i < nt) out[t0 + i] = sm[pad32(i)];
  }
  if (t0 + kScanTile >= n && threadIdx.x == kScanThreads - 1)
    out[n] = s_prefix + tot;
}

__global__ void k_scan_empty(int* out) {
  HF_PDL_ENTRY(); out[0] = 0; }

size_t scan_ws_ints(long long n) { return (size_t)ceil_div(n > 0 ? n : 1, kScanTile) + 2; }

void exclusive_scan(const int* in, int* out, long long n, int* ws, cudaStream_t s) {
  if (n <= 0) {
    HF_LAUNCH(k_scan_empty, 1, 1, 0, s, out);
    return;
  }
  int nb = (int)ceil_div(n, kScanTile);
  cudaMemsetAsync(ws, 0, sizeof(int) * (nb + 1), s);
  HF_LAUNCH(k_scan_lookback, nb, kScanThreads, 0, s, in, n, out, ws + nb, ws);
}

}  // namespace hf

extern "C" {

const char* hifuse_status_string(hifuse_status s) {
  switch (s) {
    case HIFUSE_OK: return "ok";
    case HIFUSE_ERR_INVALID_ARG: return "invalid argument";
    case HIFUSE_ERR_ALIGNMENT: return "pointer not 16-byte aligned";
    case HIFUSE_ERR_UNSUPPORTED: return "unsupported size or mode";
    case HIFUSE_ERR_WORKSPACE: return "workspace too small";
    case HIFUSE_ERR_CUDA: return "CUDA launch failed";
  }
  return "unknown status";
}

hifuse_status hifuse_read_status(const int32_t* d_status, hifuse_stream_t stream, int32_t* out_h) {
  if (!d_status || !out_h) return HIFUSE_ERR_INVALID_ARG;
  if (cudaMemcpyAsync(out_h, d_status, sizeof(int32_t), cudaMemcpyDeviceToHost, hf::st(stream)) !=
      cudaSuccess)
    return HIFUSE_ERR_CUDA;
  return cudaStreamSynchronize(hf::st(stream)) == cudaSuccess ? HIFUSE_OK : HIFUSE_ERR_CUDA;
}

int64_t hifuse_kernel_launches(void) { return hf::g_launches.load(); }

}  // extern "C"

extern "C" {

hifuse_status hifuse_stream_attach(hifuse_stream_t stream) {
  cudaStreamCaptureStatus cs;
  cudaStream_t s = hf::st(stream);
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) return HIFUSE_ERR_CUDA;
  if (cs != cudaStreamCaptureStatusNone) return HIFUSE_ERR_INVALID_ARG;
  return hf::stream_ctx(s) ? HIFUSE_OK : HIFUSE_ERR_CUDA;
}

hifuse_status hifuse_stream_release(hifuse_stream_t stream) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HIFUSE_ERR_CUDA;
  hf::StreamCtx* c = nullptr;
  {
    std::lock_guard<std::mutex> lk(hf::g_mu);
    auto it = hf::g_ctx.find(hf::StreamKey{dev, hf::st(stream)});
    if (it == hf::g_ctx.end()) return HIFUSE_OK;
    c = it->second;
    hf::g_ctx.erase(it);
  }
  if (c->ok) {
    for (int i = 0; i < hf::kBranches; i++) {
      cudaStreamSynchronize(c->br[i].side);
      cudaStreamDestroy(c->br[i].side);
      cudaEventDestroy(c->br[i].fork);
      cudaEventDestroy(c->br[i].join);
    }
    cudaEventDestroy(c->fold);
  }
  delete c;
  return HIFUSE_OK;
}

}  // extern "C"

// common.cuh -- shared device/host helpers of libhifuse (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include "hifuse.h"

#define HF_MAX_T 64
#define HF_MAX_R 256

namespace hf {

extern std::atomic<int64_t> g_launches;

inline cudaStream_t st(hifuse_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Host-derived metadata of one layer, passed by value to kernels (kernel
// parameter space is 32 KB on sm_70+ with CUDA >= 12.1; this is ~6 KB).
struct LayerMeta {
  int T, R;
  int rows;            // sum_r n_dst(t(r))
  int S;               // sum_r n_src(s(r))
  int N;               // edges
  int src_rows;        // sum_t n_src
  int dst_rows;        // sum_t n_dst
  int rel_src[HF_MAX_R];
  int rel_dst[HF_MAX_R];
  int rel_row_off[HF_MAX_R + 1];
  int slot_off[HF_MAX_R + 1];
  int n_src[HF_MAX_T];
  int n_dst[HF_MAX_T];
  int type_src_off[HF_MAX_T + 1];
  int type_dst_off[HF_MAX_T + 1];
};

// Fills `m` from a public shape; returns HIFUSE_OK or an error code.
hifuse_status make_meta(const hifuse_layer_shape* s, LayerMeta* m);

inline hifuse_status last_cuda() {
  return cudaGetLastError() == cudaSuccess ? HIFUSE_OK : HIFUSE_ERR_CUDA;
}

template <typename T>
inline T* carve(char*& p, size_t n) {
  T* r = reinterpret_cast<T*>(p);
  size_t b = (n * sizeof(T) + 255) & ~size_t(255);
  p += b;
  return r;
}
inline size_t carve_bytes(size_t n, size_t elt) { return (n * elt + 255) & ~size_t(255); }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

inline unsigned ceil_div(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

inline bool grid_nonempty(long long g) { return g > 0; }
inline bool grid_nonempty(dim3 g) { return g.x > 0 && g.y > 0 && g.z > 0; }

// Programmatic dependent launch (PDL): every kernel is launched with
// programmatic stream serialisation and begins with HF_PDL_ENTRY(): it waits
// for the previous kernel of its stream to complete (griddepcontrol.wait,
// before ANY global memory access) and then lets the next one launch
// (griddepcontrol.launch_dependents).  The next kernel's CTAs are thereby
// dispatched while this one runs, so a chain of short dependent kernels (the
// latency-bound steps of a mini-batch) loses the launch/dispatch gap at every
// boundary; correctness is that of plain stream order (each kernel still
// starts its work after its predecessor's completion and memory flush).
// Inside CUDA graphs the edges become programmatic edges.
#ifndef HF_PDL
#define HF_PDL 1
#endif
#define HF_PDL_ENTRY()                                                         \
  do {                                                                         \
    asm volatile("griddepcontrol.wait;" ::: "memory");                         \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");            \
  } while (0)

inline dim3 to_dim3(dim3 g) { return g; }
inline dim3 to_dim3(long long g) { return dim3((unsigned)g); }

template <typename... KP, typename... A>
inline void launch_k(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     A&&... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = HF_PDL ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, static_cast<A&&>(a)...);
}

#define HF_LAUNCH(kernel, grid, block, smem, stream, ...)                      \
  do {                                                                         \
    if (hf::grid_nonempty(grid)) {                                             \
      hf::launch_k(kernel, hf::to_dim3(grid), hf::to_dim3(block), (smem), (stream), \
                   __VA_ARGS__);                                               \
      hf::g_launches.fetch_add(1, std::memory_order_relaxed);                  \
    }                                                                          \
  } while (0)

// ---------------------------------------------------------------- device ---
__device__ __forceinline__ int upper_bound_i(const int* a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Fork/join of one call's independent kernels onto an auxiliary stream:
// record `fork` on the caller's stream, run the branch on `side`, record
// `join` there and make the caller's stream wait for it.  Works eagerly and
// under CUDA-graph capture (the branch becomes a parallel graph path).  The
// side streams and events belong to the caller's stream (StreamCtx, one per
// (device, caller stream)); returns false (run serially) if they cannot be
// created.
struct Branch {
  cudaStream_t side;
  cudaEvent_t fork, join;
};
constexpr int kBranches = 4;
struct StreamCtx {
  Branch br[kBranches];
  cudaEvent_t fold;     // orders the RGAT dX term after the W a_dst fold (project.cu)
  bool ok;
};
StreamCtx* stream_ctx(cudaStream_t s);   // nullptr if the resources cannot be created
bool branch_begin(cudaStream_t main, Branch* b, int idx = 0);   // idx < kBranches
void branch_end(cudaStream_t main, const Branch& b);

// cudaFuncAttributeMaxDynamicSharedMemorySize once per (device, kernel).
void set_max_smem(const void* kernel, int bytes);
// Multiprocessor count of the current device (cached device attribute).
int sm_count();

// Device-wide exclusive scan of int32 counts (reduce-then-scan, 3 kernels).
// out[0..n] receives the exclusive prefix, out[n] = total.  ws: scan_ws_ints(n).
size_t scan_ws_ints(long long n);
void exclusive_scan(const int* in, int* out, long long n, int* ws, cudaStream_t s);

}  // namespace hf

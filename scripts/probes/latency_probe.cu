// Dependent-load latency and per-kernel floor on the B200 (context for the
// latency-bound small kernels).  chase: a pointer chain of length L in a
// buffer of `bytes` (L2-resident or not); timed with CUDA events over a CUDA
// graph of G launches.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_empty() {}
__global__ void k_chase(const int* __restrict__ nxt, int L, int* out) {
  int p = threadIdx.x * 97;
  for (int i = 0; i < L; i++) p = __ldcg(nxt + p);
  if (p == -1) out[0] = p;
}

int main() {
  const int n = 1 << 24;  // 64 MB
  std::vector<int> h(n);
  for (int i = 0; i < n; i++) h[i] = (int)((i * 2654435761u + 12345u) % n);
  int *d, *o;
  cudaMalloc(&d, n * 4);
  cudaMalloc(&o, 4);
  cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time_graph = [&](auto launch, int G) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < G; i++) launch();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    for (int r = 0; r < 5; r++) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / (5 * G);
  };
  printf("empty kernel (1 block): %.2f us per graph node\n",
         time_graph([&] { k_empty<<<1, 32, 0, s>>>(); }, 100));
  printf("empty kernel (296 blocks x 256): %.2f us\n",
         time_graph([&] { k_empty<<<296, 256, 0, s>>>(); }, 100));
  for (int L : {1, 10, 100}) {
    float t = time_graph([&] { k_chase<<<1, 32, 0, s>>>(d, L, o); }, 20);
    printf("chase L=%d (64 MB table, mostly HBM): %.2f us per kernel -> %.0f ns per load\n", L, t,
           L > 1 ? (t - time_graph([&] { k_chase<<<1, 32, 0, s>>>(d, 1, o); }, 20)) * 1e3 / (L - 1) : 0.f);
  }
  // L2-resident chain: 1 MB table
  const int m = 1 << 18;
  for (int i = 0; i < m; i++) h[i] = (int)((i * 2654435761u + 777u) % m);
  cudaMemcpy(d, h.data(), m * 4, cudaMemcpyHostToDevice);
  float t1 = time_graph([&] { k_chase<<<1, 32, 0, s>>>(d, 1, o); }, 20);
  float t100 = time_graph([&] { k_chase<<<1, 32, 0, s>>>(d, 101, o); }, 20);
  printf("chase in 1 MB (L2): %.0f ns per dependent load\n", (t100 - t1) * 1e3 / 100);
  return 0;
}

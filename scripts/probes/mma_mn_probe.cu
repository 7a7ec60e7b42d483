// Probe: one tcgen05.mma kind::tf32 M=128 N=128 K=8 with MN-major operands
// (both 128B-swizzled), three descriptor encodings; prints max error vs host.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "../../paper_2408_08490_b200/csrc/tc_common.cuh"
using namespace hf::tc;

__device__ float aval(int m, int k) { return (float)(((m * 7 + k * 3) % 5) - 2) * 0.25f; }
__device__ float bval(int n, int k) { return (float)(((n * 5 + k * 11) % 7) - 3) * 0.25f; }

// mode 0: K-major A and B (baseline); mode 1: MN-major, LBO=1024 (M-block), SBO=4096;
// mode 2: MN-major with LBO/SBO swapped
__global__ void probe(int mode, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint32_t sa = base, sb = base + 32768;
  // fill
  if (mode == 0) {
    // K-major: row m (128 B = 32 tf32 of k; only k<8 nonzero)
    for (int i = tid; i < 128 * 32; i += 128) {
      int m = i / 32, k = i % 32;
      float va = k < 8 ? aval(m, k) : 0.f, vb = k < 8 ? bval(m, k) : 0.f;
      uint32_t off = sw128_off(m, k / 4) + (k % 4) * 4;
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(sa + off), "f"(va));
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + off), "f"(vb));
    }
  } else if (mode >= 3) {
    // MN-major, SWIZZLE_128B_BASE32B: atom = 4 k-rows x 128 B (32 mn), 32-byte
    // chunks XORed with (k % 4).  mode 3: m-block 1024, k-block 512;
    // mode 4: m-block 512, k-block 2048
    uint32_t mstr = mode == 3 ? 1024 : 512, kstr = mode == 3 ? 512 : 2048;
    for (int i = tid; i < 8 * 128; i += 128) {
      int k = i / 128, m = i % 128;
      float va = aval(m, k), vb = bval(m, k);
      int inrow = (m & 31) * 4;
      uint32_t off = (m >> 5) * mstr + (k >> 2) * kstr + (k & 3) * 128 +
                     ((((inrow >> 5) ^ (k & 3)) << 5) | (inrow & 31));
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(sa + off), "f"(va));
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + off), "f"(vb));
    }
  } else {
    // MN-major: atom = 8 k-rows x 32 mn (128 B); M blocks at 1024 B, k-blocks at 4096 B
    for (int i = tid; i < 32 * 128; i += 128) {
      int k = i / 128, m = i % 128;
      float va = k < 8 ? aval(m, k) : 0.f, vb = k < 8 ? bval(m, k) : 0.f;
      uint32_t off = (m >> 5) * 1024 + (k >> 3) * 4096 + sw128_off(k & 7, (m & 31) >> 2) + (m & 3) * 4;
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(sa + off), "f"(va));
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + off), "f"(vb));
    }
  }
  if (tid == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(smem_u32(&slot), 128);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = slot;
  if (tid == 0) {
    uint64_t ad, bd;
    uint32_t id;
    if (mode == 0) { ad = sw128_desc(sa, 16, 1024); bd = sw128_desc(sb, 16, 1024); id = idesc_tf32(128, 128, 0, 0); }
    else if (mode == 1) { ad = sw128_desc(sa, 1024, 4096); bd = sw128_desc(sb, 1024, 4096); id = idesc_tf32(128, 128, 1, 1); }
    else if (mode == 2) { ad = sw128_desc(sa, 4096, 1024); bd = sw128_desc(sb, 4096, 1024); id = idesc_tf32(128, 128, 1, 1); }
    else {
      uint32_t mstr = mode == 3 ? 1024 : 512, kstr = mode == 3 ? 512 : 2048;
      ad = sw128_desc(sa, mstr, kstr); bd = sw128_desc(sb, mstr, kstr);
      ad = (ad & ~(7ull << 61)) | (1ull << 61);
      bd = (bd & ~(7ull << 61)) | (1ull << 61);
      id = idesc_tf32(128, 128, 1, 1);
    }
    mma_tf32(tmem, ad, bd, id, 0u);
    mma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  for (int c0 = 0; c0 < 128; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    for (int q = 0; q < 16; q++) out[(warp * 32 + lane) * 128 + c0 + q] = v[q];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 128);
}

static float ha(int m, int k) { return (float)(((m * 7 + k * 3) % 5) - 2) * 0.25f; }
static float hb(int n, int k) { return (float)(((n * 5 + k * 11) % 7) - 3) * 0.25f; }

int main() {
  float* d;
  cudaMalloc(&d, 128 * 128 * 4);
  static float h[128 * 128];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int mode = 0; mode < 5; mode++) {
    cudaMemset(d, 0, 128 * 128 * 4);
    probe<<<1, 128, 70000>>>(mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double err = 0, nz = 0;
    for (int m = 0; m < 128; m++)
      for (int n = 0; n < 128; n++) {
        double r = 0;
        for (int k = 0; k < 8; k++) r += ha(m, k) * hb(n, k);
        err = fmax(err, fabs(r - h[m * 128 + n]));
        nz += fabs(h[m * 128 + n]);
      }
    printf("mode %d: err %s maxerr %.4f sum|out| %.1f  out[0][0..3] %.3f %.3f %.3f %.3f\n", mode,
           cudaGetErrorString(e), err, nz, h[0], h[1], h[2], h[3]);
  }
  return 0;
}

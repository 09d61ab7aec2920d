// TMEM load throughput probe (dev tool): cycles per tcgen05.ld of 128 columns x 32 lanes per warp,
// issued as 4 x .x32, 2 x .x64 or 1 x .x128, with 4 / 8 / 16 warps per CTA (one CTA per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld_probe tmem_ld_probe.cu && ./tmem_ld_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                 "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                 "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(a));
}
__device__ __forceinline__ void ldw() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int MODE>
__global__ void probe(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot + (((uint32_t)(warp & 3) * 32) << 16) + (warp >> 2) * 128 % 512;
  uint32_t acc = 0, r[32];
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      ld32(tm + c * 32, r);
      if (MODE == 1) ldw();  // wait after each x32 (serialised)
#pragma unroll
      for (int q = 0; q < 32; q += 8) acc ^= r[q];
    }
    if (MODE == 0) ldw();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x % 32 == 0) out[blockIdx.x * 32 + warp] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
  unsigned long long* d;
  uint32_t* s;
  cudaMalloc(&d, 148 * 32 * 8);
  cudaMalloc(&s, 4);
  const int iters = 2000;
  for (int warps : {4, 8, 16}) {
    for (int mode : {0, 1}) {
      if (mode == 0) probe<0><<<148, warps * 32>>>(iters, d, s);
      else probe<1><<<148, warps * 32>>>(iters, d, s);
      cudaDeviceSynchronize();
      unsigned long long h[32];
      cudaMemcpy(h, d, 32 * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
      const double bytes = (double)warps * 32 * 128 * 4 * iters;  // per SM
      printf("warps %2d mode %s: %.1f cycles per 128-col load per warp, %.1f B/clk/SM  (%s)\n", warps,
             mode ? "wait-each-x32" : "4x32-then-wait", (double)mx / iters, bytes / mx,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

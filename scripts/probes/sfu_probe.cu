// Per-SM throughput of ex2.approx, bf16x2 packing (cvt.rn.bf16x2.f32) and both interleaved (dev tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sfu_probe sfu_probe.cu && ./sfu_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pk(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}

template <int MODE>
__global__ void probe(int iters, unsigned long long* out, float* sink) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0 || MODE == 2) {
        v[i] = ex2(v[i]);
        v[i + 1] = ex2(v[i + 1]);
      }
      if (MODE == 1 || MODE == 2) acc += pk(v[i], v[i + 1]);
      if (MODE == 3) {  // integer RNE pack on the ALU pipes
        uint32_t a = __float_as_uint(v[i]), b = __float_as_uint(v[i + 1]);
        a += 0x7fffu + ((a >> 16) & 1u);
        b += 0x7fffu + ((b >> 16) & 1u);
        acc += __byte_perm(a, b, 0x7632);
      }
    }
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  float s = acc;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  if (s == 1.2345f) sink[0] = s;
}

int main() {
  unsigned long long* d;
  float* s;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&s, 4);
  const int iters = 4000, thr = 1024;
  const char* names[4] = {"ex2 only", "cvt.bf16x2 only", "ex2 + cvt (1 cvt per 2 ex2)", "int RNE pack"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) probe<0><<<148, thr>>>(iters, d, s);
      if (mode == 1) probe<1><<<148, thr>>>(iters, d, s);
      if (mode == 2) probe<2><<<148, thr>>>(iters, d, s);
      if (mode == 3) probe<3><<<148, thr>>>(iters, d, s);
      cudaDeviceSynchronize();
    }
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)thr * iters * 16;  // elements per SM
    printf("%-30s: %.2f elements/clk/SM\n", names[mode], ops / h);
  }
  return 0;
}

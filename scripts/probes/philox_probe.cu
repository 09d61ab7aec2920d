// Throughput of the attention keep-bit generator's pieces (dev tool): Philox4x32-10 with the
// 32x32->64 products as IMAD.WIDE or as IMAD.HI + IMAD, and the 16-bit threshold compares as
// per-element compare/select or as SWAR halfword compares.  One thread per 32-bit keep word
// (4 Philox calls), 1M words (the BERT-L layer's count); all variants must agree bit for bit.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o philox_probe philox_probe.cu && ./philox_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct U4 {
  uint32_t x, y, z, w;
};

template <bool WIDE>
__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    uint32_t hi0, lo0, hi1, lo1;
    if (WIDE) {
      const uint64_t p0 = static_cast<uint64_t>(M0) * c.x, p1 = static_cast<uint64_t>(M1) * c.z;
      hi0 = p0 >> 32, lo0 = (uint32_t)p0, hi1 = p1 >> 32, lo1 = (uint32_t)p1;
    } else {
      hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x, hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    }
    U4 n{hi1 ^ c.y ^ (k0 + i * 0x9E3779B9u), lo1, hi0 ^ c.w ^ (k1 + i * 0xBB67AE85u), lo0};
    c = n;
  }
  return c;
}

template <bool SWAR>
__device__ __forceinline__ uint32_t keep8(U4 r, uint32_t t) {
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
  if (!SWAR) {
    uint32_t b = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      b |= ((w[j] & 0xffffu) >= t ? 1u : 0u) << (2 * j);
      b |= ((w[j] >> 16) >= t ? 1u : 0u) << (2 * j + 1);
    }
    return b;
  }
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t ge = __vcmpgeu2(w[j], t | (t << 16));  // 0xffff per half >= t
    s |= (ge & 0x80008000u) >> (15 - 2 * j);                // bits 2j and 16 + 2j
  }
  return (s | (s >> 15)) & 0xffu;
}

template <bool WIDE, bool SWAR>
__global__ void __launch_bounds__(128) bits_kernel(int n, uint32_t k0, uint32_t k1, uint32_t t, uint32_t* out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  uint32_t word = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    U4 ctr{(uint32_t)(idx & 15) * 4 + c, (uint32_t)(idx >> 4), 3u, 0u};
    word |= keep8<SWAR>(philox<WIDE>(ctr, k0, k1), t) << (8 * c);
  }
  out[idx] = word;
}

template <bool WIDE, bool SWAR>
float run(int n, uint32_t* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  bits_kernel<WIDE, SWAR><<<(n + 127) / 128, 128>>>(n, 0x1234u, 0x5678u, 6554u, out);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) bits_kernel<WIDE, SWAR><<<(n + 127) / 128, 128>>>(n, 0x1234u, 0x5678u, 6554u, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / 20;
}

int main() {
  const int n = 1 << 20;
  uint32_t *o[4], *h = new uint32_t[n], *h0 = new uint32_t[n];
  for (auto& p : o) cudaMalloc(&p, n * 4);
  const float t[4] = {run<true, false>(n, o[0]), run<false, false>(n, o[1]), run<true, true>(n, o[2]),
                      run<false, true>(n, o[3])};
  const char* names[4] = {"IMAD.WIDE + select", "IMAD.HI+IMAD + select", "IMAD.WIDE + SWAR", "IMAD.HI+IMAD + SWAR"};
  cudaMemcpy(h0, o[0], n * 4, cudaMemcpyDeviceToHost);
  for (int v = 0; v < 4; ++v) {
    cudaMemcpy(h, o[v], n * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; ++i) bad += h[i] != h0[i];
    printf("%-24s %7.2f us per 1M keep words (%d mismatches)\n", names[v], t[v], bad);
  }
  return 0;
}

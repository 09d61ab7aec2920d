// runtime.cu — error reporting, device queries and version of libsmpk.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "smpk_common.cuh"

namespace smpk {

static thread_local char g_last_error[1024] = "";

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return SMPK_ERR_CUDA;
  }
  return SMPK_OK;
}

int num_sms() {
  static int n[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (n[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

// SM budgets for concurrently running kernels (0 = the whole GPU): GEMMs launched on a side
// stream next to the TP exchange kernels cap their persistent grid, and the exchange kernels cap
// theirs to the SMs left over, so neither waits for the other's CTAs to retire.
static int g_sm_limit_gemm = 0, g_sm_limit_rows = 0;
static int capped(int lim) {
  const int n = num_sms();
  return (lim > 0 && lim < n) ? lim : n;
}
int gemm_sms() { return capped(g_sm_limit_gemm) & ~1; }
int row_sms() { return capped(g_sm_limit_rows); }

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMPK_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v != 0;
}

}  // namespace smpk

extern "C" int smpk_set_sm_limits(int gemm_sms, int row_sms) {
  smpk::g_sm_limit_gemm = gemm_sms > 0 ? gemm_sms : 0;
  smpk::g_sm_limit_rows = row_sms > 0 ? row_sms : 0;
  return SMPK_OK;
}

extern "C" const char* smpk_last_error(void) { return smpk::g_last_error; }

extern "C" int smpk_version(void) { return 1; }

extern "C" int smpk_device_info(int* nsm, int* cc_major, int* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    smpk::set_last_error("smpk_device_info: %s", cudaGetErrorString(e));
    return SMPK_ERR_CUDA;
  }
  if (nsm) *nsm = smpk::num_sms();
  if (cc_major) cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
  if (cc_minor) cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  return SMPK_OK;
}

namespace smpk {
__global__ void rng_next_kernel(unsigned long long* counter, unsigned long long* snapshot) {
  const unsigned long long v = *counter;
  *snapshot = v;
  *counter = v + 1ull;
}
}  // namespace smpk

extern "C" int smpk_rng_next(uint64_t* counter, uint64_t* snapshot, void* stream) {
  SMPK_REQUIRE(counter && snapshot, SMPK_ERR_BAD_ARG, "smpk_rng_next: null pointer");
  smpk::rng_next_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<unsigned long long*>(counter), reinterpret_cast<unsigned long long*>(snapshot));
  return smpk::check_launch("smpk_rng_next");
}

// ---------------------------------------------------------------------------
// Fused AdamW step on one (sharded) slice of the fp32 master parameters: reads master, grad,
// m, v (16 B / element), writes master, m, v and the bf16 model copy (14 B / element); one pass,
// 128-bit vector access.  Used by the data-parallel optimizer (dp.py; PAPER.md:765 optimizer
// state sharding).  grad_scale multiplies the gradient first (1 / data-parallel degree).
// ---------------------------------------------------------------------------
namespace smpk {
__global__ void __launch_bounds__(256) adam_step_kernel(float* __restrict__ master, bf16* __restrict__ param,
                                                        const float* __restrict__ grad, float* __restrict__ m,
                                                        float* __restrict__ v, int64_t n, float lr, float b1,
                                                        float b2, float eps, float wd, float bc1, float bc2,
                                                        float grad_scale) {
  const int64_t n4 = n / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 p = reinterpret_cast<float4*>(master)[i];
    const float4 g = reinterpret_cast<const float4*>(grad)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float pv[4] = {p.x, p.y, p.z, p.w}, gv[4] = {g.x, g.y, g.z, g.w}, mv[4] = {mm.x, mm.y, mm.z, mm.w},
          sv[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float gk = gv[k] * grad_scale;
      mv[k] = b1 * mv[k] + (1.f - b1) * gk;
      sv[k] = b2 * sv[k] + (1.f - b2) * gk * gk;
      const float upd = (mv[k] / bc1) / (sqrtf(sv[k] / bc2) + eps);
      pv[k] = pv[k] - lr * (upd + wd * pv[k]);
    }
    reinterpret_cast<float4*>(master)[i] = make_float4(pv[0], pv[1], pv[2], pv[3]);
    reinterpret_cast<float4*>(m)[i] = make_float4(mv[0], mv[1], mv[2], mv[3]);
    reinterpret_cast<float4*>(v)[i] = make_float4(sv[0], sv[1], sv[2], sv[3]);
    uint2 o;
    o.x = pack_bf16x2(pv[0], pv[1]);
    o.y = pack_bf16x2(pv[2], pv[3]);
    reinterpret_cast<uint2*>(param)[i] = o;
  }
}
}  // namespace smpk

extern "C" int smpk_adam_step(float* master, void* param_bf16, const float* grad, float* m, float* v, int64_t n,
                              float lr, float beta1, float beta2, float eps, float weight_decay, int step,
                              float grad_scale, void* stream) {
  SMPK_REQUIRE(master && param_bf16 && grad && m && v && n >= 0 && step >= 1, SMPK_ERR_BAD_ARG,
               "smpk_adam_step: bad arguments");
  SMPK_REQUIRE(n % 4 == 0 && ((reinterpret_cast<uintptr_t>(master) | reinterpret_cast<uintptr_t>(grad) |
                               reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(param_bf16) & 7) == 0,
               SMPK_ERR_BAD_ARG, "smpk_adam_step: n must be a multiple of 4 with 16-B aligned buffers");
  if (n == 0) return SMPK_OK;
  const float bc1 = 1.f - powf(beta1, (float)step), bc2 = 1.f - powf(beta2, (float)step);
  int64_t grid = (n / 4 + 255) / 256;
  const int64_t cap = (int64_t)smpk::num_sms() * 8;
  if (grid > cap) grid = cap;
  smpk::adam_step_kernel<<<(unsigned)grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      master, reinterpret_cast<smpk::bf16*>(param_bf16), grad, m, v, n, lr, beta1, beta2, eps, weight_decay, bc1, bc2,
      grad_scale);
  return smpk::check_launch("smpk_adam_step");
}

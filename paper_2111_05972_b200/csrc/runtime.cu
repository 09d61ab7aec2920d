// runtime.cu — error reporting, device queries and version of libsmpk.
#include <cstdarg>
#include <cstdio>
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

// symm.cu — symmetric (peer-mapped) memory for the fused tensor-parallel collectives.
//
// Every rank of a TP group allocates the same pool, exports a CUDA IPC handle once and
// maps all peers' pools (persistent pre-registered buffers).  The row-parallel
// GEMM epilogue stores its partial tiles straight into the owning rank's pool
// (smpk_gemm_rs), the row kernels read the T partial slots in ascending rank order and
// store allgathered rows into every peer's pool (smpk_bdr_ln_fwd_ex / smpk_ln_bwd_ex), and
// smpk_symm_barrier orders those NVLink stores between ranks: each rank advances its device-resident epoch,
// writes it into every peer's flag word (st.release.sys after a system fence) and waits until all
// peers' epochs have arrived (ld.acquire.sys), with a wall-clock timeout that reports the
// stuck peer instead of hanging.
#include <mutex>

#include "smpk_common.cuh"

namespace smpk {

// 1 + index of the peer whose signal never arrived, written by the barrier kernel into pinned,
// device-mapped host memory right before it traps: the trap makes the failure sticky (every later
// CUDA call on this context fails, so no stale peer data is ever consumed) and the host can still
// read which peer was stuck without a CUDA call (smpk_symm_timeout_peer).
static volatile unsigned long long* g_timeout_host = nullptr;
static unsigned long long* g_timeout_dev = nullptr;

static int timeout_word_init() {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    void* h = nullptr;
    err = cudaHostAlloc(&h, sizeof(unsigned long long), cudaHostAllocMapped | cudaHostAllocPortable);
    if (err != cudaSuccess) return;
    *reinterpret_cast<volatile unsigned long long*>(h) = 0;
    void* d = nullptr;
    err = cudaHostGetDevicePointer(&d, h, 0);
    if (err != cudaSuccess) return;
    g_timeout_host = reinterpret_cast<volatile unsigned long long*>(h);
    g_timeout_dev = reinterpret_cast<unsigned long long*>(d);
  });
  return err == cudaSuccess ? SMPK_OK : SMPK_ERR_CUDA;
}

// local_flags[0..31]: epoch last signalled by each peer; local_flags[32]: this rank's epoch
// counter (device-resident so graph replays advance it; every rank runs the same barrier
// sequence, so the counters stay in lockstep).
__global__ void symm_barrier_kernel(uint32_t* const* peer_flags, uint32_t* local_flags, int T, int rank,
                                    unsigned long long timeout_ns, unsigned long long* timeout_word) {
  const int t = threadIdx.x;
  const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(local_flags + 32) + 1;
  __syncwarp();
  if (t == 0) local_flags[32] = epoch;
  if (t >= T) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer_flags[t] + rank), "r"(epoch) : "memory");
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(local_flags + t) : "memory");
    if ((int32_t)(v - epoch) >= 0) break;
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > timeout_ns) {
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(timeout_word), "l"((unsigned long long)(t + 1))
                   : "memory");
      __threadfence_system();
      __trap();  // sticky: the step fails loudly instead of reading a stuck peer's stale region
    }
    __nanosleep(64);
  }
}

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

static PFN_getAddressRange get_range_fn() {
  static PFN_getAddressRange fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_getAddressRange>(p);
  });
  return fn;
}

}  // namespace smpk

using namespace smpk;

// IPC handle of the allocation containing ptr, and ptr's byte offset inside it.
extern "C" int smpk_symm_export(void* ptr, void* handle_out, int64_t* offset) {
  SMPK_REQUIRE(ptr && handle_out && offset, SMPK_ERR_BAD_ARG, "smpk_symm_export: bad arguments");
  PFN_getAddressRange fn = get_range_fn();
  SMPK_REQUIRE(fn != nullptr, SMPK_ERR_CUDA, "smpk_symm_export: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = fn(&base, &size, (CUdeviceptr)ptr);
  SMPK_REQUIRE(r == CUDA_SUCCESS, SMPK_ERR_CUDA, "smpk_symm_export: address range (%d)", (int)r);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_symm_export: %s", cudaGetErrorString(e));
  memcpy(handle_out, &h, sizeof(h));
  *offset = (int64_t)((CUdeviceptr)ptr - base);
  return SMPK_OK;
}

extern "C" int smpk_symm_barrier(void* const* peer_flags, void* local_flags, int T, int rank, double timeout_s,
                                 void* stream) {
  SMPK_REQUIRE(peer_flags && local_flags && T > 0 && T <= 32 && rank >= 0 && rank < T, SMPK_ERR_BAD_ARG,
               "smpk_symm_barrier: bad arguments");
  SMPK_REQUIRE(timeout_word_init() == SMPK_OK, SMPK_ERR_CUDA, "smpk_symm_barrier: mapped timeout word");
  symm_barrier_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint32_t* const*>(peer_flags), reinterpret_cast<uint32_t*>(local_flags), T, rank,
      (unsigned long long)(timeout_s * 1e9), g_timeout_dev);
  return check_launch("smpk_symm_barrier");
}

// 0 = no timeout so far; otherwise 1 + index of the peer whose signal never arrived.  A plain
// host read of mapped memory: valid after the barrier's trap has poisoned the CUDA context.
extern "C" int smpk_symm_timeout_peer(void) { return g_timeout_host ? (int)*g_timeout_host : 0; }

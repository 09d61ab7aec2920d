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

// ---------------------------------------------------------------------------------------------
// Mailbox copies for the overlapped TP exchanges (tp_exchange = "overlap" / "chunks").
//
// smpk_peer_put: one launch moves up to SMPK_PUT_MAX_RANGES byte ranges from local memory into
// peer-mapped slots (plain 16-byte vector stores over NVLink, a few CTAs per range: the copy runs
// as an ordinary kernel next to the other micro-batch's GEMMs -- CUDA-graph memcpy nodes of
// different branches were measured to serialise).  Ranges belong to destination groups; the last
// CTA of a group (per-group arrival counter, re-armed for the next launch) fences and raises the
// group's remote ready word; with an ack word the group first waits until the receiver released
// the slot of the previous round (ack == 0) and marks it in flight (ack = 1) when done.
// smpk_flag_wait: one thread per word spins (acquire.sys) until word == value, then re-arms it
// (0); a peer that never signals traps after the timeout (as the barrier does).
// smpk_flag_set: release-stores value into each word (e.g. the ack words of the senders).
// ---------------------------------------------------------------------------------------------
namespace smpk {

struct PutArgs {
  int nr;
  const int4* src[SMPK_PUT_MAX_RANGES];
  int4* dst[SMPK_PUT_MAX_RANGES];
  long long n16[SMPK_PUT_MAX_RANGES];
  int grp[SMPK_PUT_MAX_RANGES];
  int cta0[SMPK_PUT_MAX_RANGES + 1];
  uint32_t* ready[SMPK_PUT_MAX_GROUPS];
  uint32_t* ack[SMPK_PUT_MAX_GROUPS];
  int gctas[SMPK_PUT_MAX_GROUPS];
  uint32_t* counter;
  unsigned long long timeout_ns;
  unsigned long long* timeout_word;
};

__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void spin_until(const uint32_t* p, uint32_t want, unsigned long long timeout_ns,
                                           unsigned long long* timeout_word, int who) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_acq_sys(p) != want) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > timeout_ns) {
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(timeout_word), "l"((unsigned long long)(who + 1))
                   : "memory");
      __threadfence_system();
      __trap();
    }
    __nanosleep(32);
  }
}

__global__ void __launch_bounds__(256) peer_put_kernel(PutArgs a) {
  int r = 0;
  while (r + 1 < a.nr && (int)blockIdx.x >= a.cta0[r + 1]) ++r;
  const int g = a.grp[r];
  if (a.ack[g]) {
    if (threadIdx.x == 0) spin_until(a.ack[g], 0u, a.timeout_ns, a.timeout_word, g);
    __syncthreads();
  }
  const int4* __restrict__ s = a.src[r];
  int4* __restrict__ d = a.dst[r];
  const long long n = a.n16[r];
  const long long stride = (long long)(a.cta0[r + 1] - a.cta0[r]) * blockDim.x;
  long long i = (long long)(blockIdx.x - a.cta0[r]) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const int4 v0 = s[i], v1 = s[i + stride], v2 = s[i + 2 * stride], v3 = s[i + 3 * stride];
    d[i] = v0;
    d[i + stride] = v1;
    d[i + 2 * stride] = v2;
    d[i + 3 * stride] = v3;
  }
  for (; i < n; i += stride) d[i] = s[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(a.counter + g, 1u) == (uint32_t)a.gctas[g] - 1) {
    a.counter[g] = 0;  // re-armed for the next launch (kernel boundary orders it)
    __threadfence_system();
    if (a.ack[g]) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(a.ack[g]), "r"(1u) : "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.ready[g]), "r"(1u) : "memory");
  }
}

struct FlagArgs {
  int n;
  uint32_t* w[SMPK_PUT_MAX_GROUPS];
  int who[SMPK_PUT_MAX_GROUPS];
  uint32_t value;
  unsigned long long timeout_ns;
  unsigned long long* timeout_word;
};

__global__ void flag_wait_kernel(FlagArgs a) {
  const int t = threadIdx.x;
  if (t < a.n) {
    spin_until(a.w[t], a.value, a.timeout_ns, a.timeout_word, a.who[t]);
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(a.w[t]), "r"(0u) : "memory");
  }
  __threadfence();
}

__global__ void flag_set_kernel(FlagArgs a) {
  const int t = threadIdx.x;
  __threadfence_system();
  if (t < a.n) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.w[t]), "r"(a.value) : "memory");
}

static int put_ctas() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMPK_PUT_CTAS");
    v = e ? atoi(e) : 32;
    if (v < 1) v = 1;
  }
  return v;
}

}  // namespace smpk

extern "C" int smpk_peer_put(const smpk_put_range* ranges, int nr, const smpk_put_group* groups, int ng,
                             void* counter, double timeout_s, void* stream) {
  SMPK_REQUIRE(ranges && groups && counter && nr >= 1 && nr <= SMPK_PUT_MAX_RANGES && ng >= 1 &&
                   ng <= SMPK_PUT_MAX_GROUPS,
               SMPK_ERR_BAD_ARG, "smpk_peer_put: bad arguments (nr %d, ng %d)", nr, ng);
  SMPK_REQUIRE(timeout_word_init() == SMPK_OK, SMPK_ERR_CUDA, "smpk_peer_put: mapped timeout word");
  PutArgs a;
  memset(&a, 0, sizeof(a));
  a.nr = nr;
  int64_t total = 0;
  for (int r = 0; r < nr; ++r) {
    const smpk_put_range& q = ranges[r];
    SMPK_REQUIRE(q.src && q.dst && q.bytes > 0 && q.bytes % 16 == 0 && q.group >= 0 && q.group < ng &&
                     ((uintptr_t)q.src % 16) == 0 && ((uintptr_t)q.dst % 16) == 0,
                 SMPK_ERR_BAD_ARG, "smpk_peer_put: range %d must be 16-byte aligned and sized", r);
    total += q.bytes;
  }
  for (int g = 0; g < ng; ++g) {
    SMPK_REQUIRE(groups[g].ready != nullptr, SMPK_ERR_BAD_ARG, "smpk_peer_put: group %d has no ready word", g);
    a.ready[g] = groups[g].ready;
    a.ack[g] = groups[g].ack;
  }
  const int budget = put_ctas();
  int cta = 0;
  for (int r = 0; r < nr; ++r) {
    int c = (int)((double)budget * (double)ranges[r].bytes / (double)total + 0.5);
    if (c < 1) c = 1;
    a.src[r] = reinterpret_cast<const int4*>(ranges[r].src);
    a.dst[r] = reinterpret_cast<int4*>(ranges[r].dst);
    a.n16[r] = ranges[r].bytes / 16;
    a.grp[r] = ranges[r].group;
    a.cta0[r] = cta;
    a.gctas[ranges[r].group] += c;
    cta += c;
  }
  a.cta0[nr] = cta;
  a.counter = reinterpret_cast<uint32_t*>(counter);
  a.timeout_ns = (unsigned long long)(timeout_s * 1e9);
  a.timeout_word = g_timeout_dev;
  peer_put_kernel<<<cta, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return check_launch("smpk_peer_put");
}

static int flag_launch(void* const* words, const int* who, int n, uint32_t value, double timeout_s, void* stream,
                       bool wait) {
  SMPK_REQUIRE(words && n >= 1 && n <= SMPK_PUT_MAX_GROUPS, SMPK_ERR_BAD_ARG, "smpk_flag_%s: bad arguments",
               wait ? "wait" : "set");
  SMPK_REQUIRE(timeout_word_init() == SMPK_OK, SMPK_ERR_CUDA, "smpk_flag: mapped timeout word");
  FlagArgs a;
  memset(&a, 0, sizeof(a));
  a.n = n;
  for (int i = 0; i < n; ++i) {
    a.w[i] = reinterpret_cast<uint32_t*>(words[i]);
    a.who[i] = who ? who[i] : i;
  }
  a.value = value;
  a.timeout_ns = (unsigned long long)(timeout_s * 1e9);
  a.timeout_word = g_timeout_dev;
  if (wait) flag_wait_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  else flag_set_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return check_launch(wait ? "smpk_flag_wait" : "smpk_flag_set");
}

extern "C" int smpk_flag_wait(void* const* words, const int* who, int n, uint32_t value, double timeout_s,
                              void* stream) {
  return flag_launch(words, who, n, value, timeout_s, stream, true);
}

extern "C" int smpk_flag_set(void* const* words, int n, uint32_t value, void* stream) {
  return flag_launch(words, nullptr, n, value, 0.0, stream, false);
}

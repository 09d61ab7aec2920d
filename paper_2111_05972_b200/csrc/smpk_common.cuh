// smpk_common.cuh — shared device helpers for the sm_100a kernels of libsmpk.
//
// Inline-PTX wrappers for mbarrier, TMA (cp.async.bulk.tensor), tcgen05 (MMA,
// TMEM alloc/ld, commit) plus the bf16 / Philox helpers every kernel uses.
// Written for -gencode arch=compute_100a,code=sm_100a only.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "smpk.h"

namespace smpk {

using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------------------
// error plumbing (host)
// ---------------------------------------------------------------------------
void set_last_error(const char* fmt, ...);
int check_launch(const char* what);

#define SMPK_REQUIRE(cond, code, ...)       \
  do {                                      \
    if (!(cond)) {                          \
      ::smpk::set_last_error(__VA_ARGS__);  \
      return (code);                        \
    }                                       \
  } while (0)

int num_sms();
int gemm_sms();  // num_sms() under smpk_set_sm_limits (even)
int row_sms();
bool pdl_enabled();  // SMPK_PDL=0 turns programmatic dependent launch off (A/B)

// ---------------------------------------------------------------------------
// programmatic dependent launch: a kernel launched with launch_pdl may be scheduled while the
// previous kernel on its stream is still finishing.  Every such kernel acquires its on-chip
// resources (barriers, TMEM), then calls pdl_trigger() (its own dependents may now be scheduled:
// all of its CTAs are resident or done and hold what they need, so they cannot starve) and
// pdl_wait() (returns once the previous grid completed and its writes are visible) BEFORE its
// first global-memory access.  Both are no-ops for a kernel launched without the attribute.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------------------
// shared-memory / mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// try_wait with a suspend-time hint: a waiting warp sleeps in the barrier unit instead of
// re-issuing the probe loop (the spin loops were ~1/3 of the issued instructions of the
// attention backward in ncu).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)
      : "memory");
}

// non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// ---------------------------------------------------------------------------
// TMA
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// 1-D bulk copy global -> shared (bytes % 16 == 0, 16-B aligned), completes on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// tcgen05 / TMEM
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 in, fp32 accumulate; one thread issues.
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05 ops of this thread finish.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// ---- CTA pair (cta_group::2): two CTAs of a cluster on one TPC share one M=256 MMA ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// TMA load issued by either CTA of the pair; the transaction bytes complete on the LEADER's
// (rank 0) barrier at the same shared offset (clearing the peer bit of the cluster address).
__device__ __forceinline__ void tma_load_4d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 int c2, int c3) {
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
      : "memory");
}

__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// completion of the pair's prior MMAs arrives on the barrier at this offset in every CTA of mask
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// arrive (release, cluster scope) on the barrier at this offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// Remote arrive without release semantics: for handing a TMEM buffer back (the tcgen05.ld reads
// are ordered by tcgen05.wait::ld + fence::before_thread_sync, not by memory).  The release
// form costs a MEMBAR.ALL.GPU per arriving warp (ncu: ~8% of the GEMM epilogue's stall samples).
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// local arrive, relaxed (see above)
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 32 lanes x 32 consecutive fp32 columns: thread t receives lane (base_lane + t).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// make generic-proxy shared-memory writes visible to the async proxy (tcgen05.mma / TMA)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// true in exactly one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
      "elect.sync rx|px, 0xffffffff;\n\t"
      "@px mov.s32 %0, 1;\n\t}"
      : "+r"(pred));
  return pred != 0;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void named_barrier_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// byte offset of 16-B granule g (0..7) of row r inside a K-major SWIZZLE_128B tile
// (8-row x 128-B atoms stacked every 1024 B): the hardware XORs the granule with r % 8.
__device__ __forceinline__ uint32_t sw128_offset(int r, int g) {
  return static_cast<uint32_t>((r >> 3) * 1024 + (r & 7) * 128 + ((g ^ (r & 7)) << 4));
}

// UMMA shared-memory descriptor (sm_100 "version 1"), SWIZZLE_128B layout.
//   K-major : 8-row x 128B swizzle atoms stacked every `sbo` bytes (LBO unused -> 1).
//   MN-major: 64-element MN chunks every `lbo` bytes, 8-deep K groups every `sbo` bytes.
__device__ __forceinline__ uint64_t make_sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // descriptor version for tcgen05
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::f16, A/B = bf16, D = fp32, dense.
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N, bool a_mn_major, bool b_mn_major) {
  return (1u << 4)                                   // D format f32
         | (1u << 7)                                 // A format bf16
         | (1u << 10)                                // B format bf16
         | (static_cast<uint32_t>(a_mn_major) << 15)  // A major
         | (static_cast<uint32_t>(b_mn_major) << 16)  // B major
         | (static_cast<uint32_t>(N >> 3) << 17)      //
         | (static_cast<uint32_t>(M >> 4) << 24);
}

// ---------------------------------------------------------------------------
// numerics
// ---------------------------------------------------------------------------
__device__ __forceinline__ float bf2f(bf16 v) { return __bfloat162float(v); }
__device__ __forceinline__ bf16 f2bf(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float2 unpack_bf16x2(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(v);
}

// Dropout keep bits applied to packed bf16 pairs with two instructions per pair (one PRMT, one
// AND) instead of a bit test and a select per element.  sh[s] = w << s for s = 0..7 puts bit
// 8k+u of w at the sign bit of byte k of sh[7-u]; PRMT's sign-replicate selectors spread that
// bit over a 16-bit half.  keep_pair_mask(sh, k, u) (u even, k, u compile-time) is 0xffff in the
// low half iff bit 8k+u is set and 0xffff0000 iff bit 8k+u+1 is set.
__device__ __forceinline__ void keep_shifts(uint32_t w, uint32_t (&sh)[8]) {
#pragma unroll
  for (int s = 0; s < 8; ++s) sh[s] = w << s;
}
__device__ __forceinline__ uint32_t keep_pair_mask(const uint32_t (&sh)[8], int k, int u) {
  const uint32_t sel = ((0xCu + k) << 12) | ((0xCu + k) << 8) | ((0x8u + k) << 4) | (0x8u + k);
  uint32_t m;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(m) : "r"(sh[7 - u]), "r"(sh[6 - u]), "r"(sel));
  return m;
}

// bf16 round-to-nearest-even kept in fp32, with integer ops (keeps the XU pipe free).
__device__ __forceinline__ float round_bf16(float v) {
  uint32_t u = __float_as_uint(v);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return __uint_as_float(u & 0xFFFF0000u);
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Standard normal CDF Phi(z) = 0.5 (1 + erf(z/sqrt2)) with erf from Abramowitz & Stegun
// 7.1.26 (|err| <= 1.5e-7) written for the epilogue issue budget: one rcp.approx and one
// ex2.approx (no range fix-ups), the 1/sqrt2, log2(e) and the final 1/2 folded into the
// constants.  With x = |z|/sqrt2:  t = 1/(1 + p x),  q = 0.5 poly(t) exp(-x^2),
// Phi = 1 - q (z >= 0) or q (z < 0).  Also returns e = exp(-z^2/2) for the density.
__device__ __forceinline__ float normal_cdf(float z, float& e) {
  const float t = rcp_approx(fmaf(fabsf(z), 0.23164188f /* p / sqrt2 */, 1.f));
  e = ex2_approx((z * -0.72134752f /* -log2(e)/2 */) * z);
  const float ph =
      t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 0.5307027145f, -0.7265760135f), 0.7107068705f), -0.142248368f),
               0.127414796f);  // 0.5 * A&S a1..a5
  const float q = ph * e;
  return z >= 0.f ? 1.f - q : q;
}

// Activation functions. act: SMPK_ACT_GELU_ERF / SMPK_ACT_GELU_TANH / SMPK_ACT_RELU.
__device__ __forceinline__ float act_fwd(int act, float z) {
  if (act == SMPK_ACT_RELU) return z > 0.f ? z : 0.f;
  if (act == SMPK_ACT_GELU_TANH) {
    // 0.5 z (1 + tanh(k0 (z + k1 z^3))) with k0 folded: u = z (k0 + k0 k1 z^2)
    const float u = z * fmaf(z * z, 0.0356774081f, 0.7978845608f);
    const float hz = 0.5f * z;
    return fmaf(hz, tanh_approx(u), hz);
  }
  float e;
  return z * normal_cdf(z, e);
}

__device__ __forceinline__ float act_bwd(int act, float z) {  // d act / dz
  if (act == SMPK_ACT_RELU) return z > 0.f ? 1.f : 0.f;
  if (act == SMPK_ACT_GELU_TANH) {
    const float z2 = z * z;
    const float u = z * fmaf(z2, 0.0356774081f, 0.7978845608f);
    const float t = tanh_approx(u);
    // 0.5 (1 + t) + 0.5 z (1 - t^2) k0 (1 + 3 k1 z^2)
    const float du = fmaf(z2, 0.1070322243f, 0.7978845608f);  // k0 (1 + 3 k1 z^2)
    return fmaf(0.5f * z * du, fmaf(-t, t, 1.f), fmaf(0.5f, t, 0.5f));
  }
  float e;
  const float cdf = normal_cdf(z, e);
  return fmaf(z * 0.3989422804014327f, e, cdf);
}

// Paired forms of normal_cdf / act_fwd / act_bwd for (even, odd) column pairs: the same operation
// sequence per lane (bit-identical results) with the fp32 arithmetic as FFMA2 / FMUL2, so an
// epilogue warp issues half the FMA-pipe instructions (the GEMM epilogue is issue-heavy).
__device__ __forceinline__ float2 f2c(float c) { return make_float2(c, c); }
__device__ __forceinline__ float2 normal_cdf2(float2 z, float2& e) {
  const float2 den = __ffma2_rn(make_float2(fabsf(z.x), fabsf(z.y)), f2c(0.23164188f), f2c(1.f));
  const float2 t = make_float2(rcp_approx(den.x), rcp_approx(den.y));
  const float2 zz = __fmul2_rn(__fmul2_rn(z, f2c(-0.72134752f)), z);
  e = make_float2(ex2_approx(zz.x), ex2_approx(zz.y));
  float2 p = __ffma2_rn(t, f2c(0.5307027145f), f2c(-0.7265760135f));
  p = __ffma2_rn(t, p, f2c(0.7107068705f));
  p = __ffma2_rn(t, p, f2c(-0.142248368f));
  p = __ffma2_rn(t, p, f2c(0.127414796f));
  const float2 q = __fmul2_rn(__fmul2_rn(t, p), e);
  return make_float2(z.x >= 0.f ? 1.f - q.x : q.x, z.y >= 0.f ? 1.f - q.y : q.y);
}
__device__ __forceinline__ float2 act_fwd2(int act, float2 z) {
  if (act == SMPK_ACT_RELU) return make_float2(z.x > 0.f ? z.x : 0.f, z.y > 0.f ? z.y : 0.f);
  if (act == SMPK_ACT_GELU_TANH) {
    const float2 u = __fmul2_rn(z, __ffma2_rn(__fmul2_rn(z, z), f2c(0.0356774081f), f2c(0.7978845608f)));
    const float2 hz = __fmul2_rn(f2c(0.5f), z);
    return __ffma2_rn(hz, make_float2(tanh_approx(u.x), tanh_approx(u.y)), hz);
  }
  float2 e;
  return __fmul2_rn(z, normal_cdf2(z, e));
}
__device__ __forceinline__ float2 act_bwd2(int act, float2 z) {
  if (act == SMPK_ACT_RELU) return make_float2(z.x > 0.f ? 1.f : 0.f, z.y > 0.f ? 1.f : 0.f);
  if (act == SMPK_ACT_GELU_TANH) {
    const float2 z2 = __fmul2_rn(z, z);
    const float2 u = __fmul2_rn(z, __ffma2_rn(z2, f2c(0.0356774081f), f2c(0.7978845608f)));
    const float2 t = make_float2(tanh_approx(u.x), tanh_approx(u.y));
    const float2 du = __ffma2_rn(z2, f2c(0.1070322243f), f2c(0.7978845608f));
    return __ffma2_rn(__fmul2_rn(__fmul2_rn(f2c(0.5f), z), du), __ffma2_rn(make_float2(-t.x, -t.y), t, f2c(1.f)),
                      __ffma2_rn(f2c(0.5f), t, f2c(0.5f)));
  }
  float2 e;
  const float2 cdf = normal_cdf2(z, e);
  return __ffma2_rn(__fmul2_rn(z, f2c(0.3989422804014327f)), e, cdf);
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (counter-based; reproduced bit-exactly by oracle/philox.py)
// ---------------------------------------------------------------------------
struct u32x4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    uint64_t p0 = static_cast<uint64_t>(M0) * c.x;
    uint64_t p1 = static_cast<uint64_t>(M1) * c.z;
    uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    u32x4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// Round keys of one Philox key, computed once when a thread makes several calls with it.
struct PhiloxRoundKeys {
  uint32_t k0[10], k1[10];
};
__host__ __device__ __forceinline__ PhiloxRoundKeys philox_round_keys(uint32_t k0, uint32_t k1) {
  PhiloxRoundKeys r;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    r.k0[i] = k0 + static_cast<uint32_t>(i) * 0x9E3779B9u;
    r.k1[i] = k1 + static_cast<uint32_t>(i) * 0xBB67AE85u;
  }
  return r;
}
__host__ __device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, const PhiloxRoundKeys& rk) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint64_t p0 = static_cast<uint64_t>(M0) * c.x;
    const uint64_t p1 = static_cast<uint64_t>(M1) * c.z;
    u32x4 n;
    n.x = static_cast<uint32_t>(p1 >> 32) ^ c.y ^ rk.k0[i];
    n.y = static_cast<uint32_t>(p1);
    n.z = static_cast<uint32_t>(p0 >> 32) ^ c.w ^ rk.k1[i];
    n.w = static_cast<uint32_t>(p0);
    c = n;
  }
  return c;
}

// Dropout draws 16 bits per element: one Philox call covers 8 consecutive columns.
//   counter = (col >> 3, row, layer, site); word = out[(col >> 1) & 3];
//   u16 = (word >> (16 * (col & 1))) & 0xffff;  keep iff u16 >= rint(p * 65536)
__host__ __device__ __forceinline__ uint32_t dropout_threshold(float p) {
  return static_cast<uint32_t>(rintf(p * 65536.f));
}

// Philox key of one training step: the host seed plus the device-resident step word times the
// 64-bit golden ratio (rng_step may be null: key = seed).  The step word is snapshotted per
// top-level forward (smpk_rng_next), so CUDA-graph replays and consecutive steps draw new masks
// while a layer's backward re-reads the value its forward used (oracle/philox.py step_key).
__device__ __forceinline__ uint64_t philox_key(uint64_t seed, const uint64_t* rng_step) {
  return rng_step ? seed + __ldg(reinterpret_cast<const unsigned long long*>(rng_step)) * 0x9E3779B97F4A7C15ull
                  : seed;
}

// keep flags for 8 consecutive columns (precomputed round keys of the step key)
__device__ __forceinline__ uint32_t dropout_keep8_bits(const PhiloxRoundKeys& rk, uint32_t layer, uint32_t site,
                                                       uint64_t g, int col0, uint32_t thresh) {
  u32x4 c = {static_cast<uint32_t>(col0 >> 3), static_cast<uint32_t>(g), layer, site};
  u32x4 r = philox4x32_10(c, rk);
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    bits |= ((w[j] & 0xffffu) >= thresh ? 1u : 0u) << (2 * j);
    bits |= ((w[j] >> 16) >= thresh ? 1u : 0u) << (2 * j + 1);
  }
  return bits;
}

// keep flags for 8 consecutive columns col0..col0+7 (col0 % 8 == 0) of logical row g
__device__ __forceinline__ void dropout_keep8(uint64_t seed, uint32_t layer, uint32_t site, uint64_t g, int col0,
                                              uint32_t thresh, bool (&keep)[8]) {
  u32x4 c = {static_cast<uint32_t>(col0 >> 3), static_cast<uint32_t>(g), layer, site};
  u32x4 r = philox4x32_10(c, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    keep[2 * j] = (w[j] & 0xffffu) >= thresh;
    keep[2 * j + 1] = (w[j] >> 16) >= thresh;
  }
}


// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: set once per (kernel, device).
template <typename Kern>
inline cudaError_t smem_attr_once(Kern kern, int bytes, unsigned long long& done_mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  if ((done_mask >> dev) & 1ull) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done_mask |= 1ull << dev;
  return e;
}

}  // namespace smpk

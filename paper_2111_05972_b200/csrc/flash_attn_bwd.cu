// flash_attn_bwd.cu — fused attention backward on tcgen05/TMEM/TMA (sm_100a).
//
// CTA = (128-key tile j, local head, sample); it keeps K_j, V_j in smem and the dK, dV
// accumulators in TMEM while streaming the query tiles i (i >= j when causal).  One TMEM
// region A (128 columns) is reused three times per query tile:
//   (a) S^T  = K_j Q_i^T  -> A          (M=keys, N=queries, K=dh)
//       softmax-backward warps (thread = key row): P = exp2(S*scale*log2e + mask - lse2[q])
//       (recomputed, never stored in HBM), kept in registers as bf16; Pd^T = keep ? P : 0
//       -> smem (K-major A operand)
//   (b) dV += Pd^T dO_i,  dP^T = V_j dO_i^T -> A
//       dS^T = P * (keep ? dP/(1-p) : 0  - Delta[q]) -> smem (same buffer: dV has read Pd^T)
//   (c) dK += dS^T Q_i,  dQ_i(j) = dS K_j -> A (M=queries), drained as an fp32 partial per key
//       tile; smpk_flash_dq_reduce sums the partials in key-tile order (bit-deterministic).
// 1/(1-p) of dV and the softmax scale of dK / dQ are applied once at the end.  The small
// footprint (256 TMEM columns, ~100 KB smem at dh=64) lets two CTAs share an SM, so one
// CTA's softmax work overlaps the other's tensor-core work.
// Dropout keep bits (smpk_attn_dropout_bits, shared with the forward) arrive by TMA as a
// [128 queries x 4 words] tile and are read column-wise (bit = key).
#include <cstring>

#include "smpk_common.cuh"

namespace smpk {

int make_tma_4d(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int nb1, int64_t s1,
                int nb2, int64_t s2, int box_inner, int box_outer, const char* name);
int make_tma_4d_b32(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                    int box_outer, const char* name);
int make_tma_4d_f32sw(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                      int box_outer, const char* name);

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(0), "r"(0)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(0), "r"(0)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int FB_THREADS = 256;

struct FaBwdArgs {
  int B, nh, s;
  const float* lse;    // [B, nh, s] log2 domain (from the forward)
  const float* delta;  // [B, nh, s] rowsum(dO * O)
  const float* mask;   // [B, s] additive or null
  float scale_log2, scale;
  int causal;
  int dropout;
  float inv_keep;
  bf16* dqkv;
  int64_t ld;  // of qkv / dqkv
  int64_t H;   // nh * dh
  float* dq_part;  // [n_kt][B*s][H] (v1 kernel)
  int trace;
  int* dq_cnt;     // [B][nh][n_qt] contributors of each query tile's dQ so far (zeroed by the delta kernel)
};

template <int DH>
struct FaBwdCfg {
  static constexpr int TILE = 128 * DH * 2;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + TILE;
  static constexpr int OFF_Q = OFF_V + TILE;
  static constexpr int OFF_DO = OFF_Q + TILE;
  static constexpr int OFF_PS = OFF_DO + TILE;  // Pd^T, then dS^T (128 x 128 bf16)
  static constexpr int OFF_LSE = OFF_PS + 32768;
  static constexpr int OFF_DELTA = OFF_LSE + 512;
  static constexpr int OFF_BITS = OFF_DELTA + 512;  // [128 queries][4 words]
  static constexpr int OFF_KBT = OFF_BITS + 2048;   // the same bits transposed [4 words][128 queries]
  static constexpr int OFF_BAR = OFF_KBT + 2048;
  static constexpr int SMEM = 1024 + OFF_BAR + 256;
  // TMEM: A [0,128) (S^T -> dP^T -> dQ), dV [128, 128+DH), dK [128+DH, 128+2DH)
  static constexpr uint32_t TMEM_COLS = DH == 64 ? 256 : 512;
  static constexpr int QDO_BYTES = 2 * TILE + 1024 + 2048;
};

template <int DH>
__global__ void __launch_bounds__(FB_THREADS, (DH == 64 ? 2 : 1))
    flash_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                     const __grid_constant__ CUtensorMap tmBits, const FaBwdArgs a) {
  using Cfg = FaBwdCfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ array (not an integer round trip) keeps the shared
  // address space visible to the compiler: LDS / STS instead of generic LD / ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* qdo_full = bar + 1;
  uint64_t* qdo_empty = bar + 2;
  uint64_t* s_full = bar + 3;
  uint64_t* p_full = bar + 4;
  uint64_t* dp_full = bar + 5;
  uint64_t* ds_full = bar + 6;
  uint64_t* dq_full = bar + 7;
  uint64_t* a_free = bar + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_kt = a.s / 128;
  const int j = (int)blockIdx.x;  // key tile
  const int h = blockIdx.y, b = blockIdx.z;
  const int i0 = a.causal ? j : 0;
  const int nt = n_kt - i0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmDO);
    if (a.dropout) tma_prefetch_desc(&tmBits);
    mbar_init(kv_full, 1);
    mbar_init(qdo_full, 1);
    mbar_init(qdo_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);  // one arrive per softmax warp
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 4);
    mbar_init(dq_full, 1);
    mbar_init(a_free, 4);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tA = tmem, tdV = tmem + 128, tdK = tmem + 128 + DH;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_arrive_expect_tx(kv_full, 2 * Cfg::TILE);
#pragma unroll
      for (int c = 0; c < DH / 64; ++c) {
        tma_load_4d(smem + Cfg::OFF_K + c * 16384, &tmK, kv_full, c * 64, j * 128, h, b);
        tma_load_4d(smem + Cfg::OFF_V + c * 16384, &tmV, kv_full, c * 64, j * 128, h, b);
      }
      const int64_t bh_row = ((int64_t)b * a.nh + h) * a.s;
      for (int t = 0; t < nt; ++t) {
        const int i = i0 + t;
        // dO, lse, Delta and the keep bits of tile t are loaded as soon as tile t-1's dS pass has
        // read them (ds_full: after the dV / dP^T MMAs and the softmax warps' last use), i.e. while
        // tile t-1's dK / dQ MMAs and dQ drain still run; Q waits for those MMAs (qdo_empty).
        if (t > 0) mbar_wait(ds_full, (t - 1) & 1);
        mbar_arrive_expect_tx(qdo_full, 2 * Cfg::TILE + 1024 + (a.dropout ? 2048 : 0));
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
          tma_load_4d(smem + Cfg::OFF_DO + c * 16384, &tmDO, qdo_full, c * 64, i * 128, h, b);
        const int64_t off = bh_row + (int64_t)i * 128;
        bulk_load(smem + Cfg::OFF_LSE, a.lse + off, 512, qdo_full);
        bulk_load(smem + Cfg::OFF_DELTA, a.delta + off, 512, qdo_full);
        if (a.dropout) tma_load_4d(smem + Cfg::OFF_BITS, &tmBits, qdo_full, j * 4, (int)off, 0, 0);
        mbar_wait(qdo_empty, (t & 1) ^ 1);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
          tma_load_4d(smem + Cfg::OFF_Q + c * 16384, &tmQ, qdo_full, c * 64, i * 128, h, b);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp; one elected lane issues) ----------------
    const uint32_t idKK = make_idesc_bf16(128, 128, false, false);
    const uint32_t idKM = make_idesc_bf16(128, DH, false, true);
    const uint32_t idMM = make_idesc_bf16(128, DH, true, true);
    const uint32_t k_base = smem_u32(smem + Cfg::OFF_K), v_base = smem_u32(smem + Cfg::OFF_V);
    const uint32_t q_base = smem_u32(smem + Cfg::OFF_Q), do_base = smem_u32(smem + Cfg::OFF_DO);
    const uint32_t ps = smem_u32(smem + Cfg::OFF_PS);
    mbar_wait(kv_full, 0);
    for (int t = 0; t < nt; ++t) {
      mbar_wait(qdo_full, t & 1);
      if (t > 0) mbar_wait(a_free, (t - 1) & 1);  // dQ_{t-1} drained: region A free
      tc_fence_after();
      if (elect_one()) {  // (a) S^T = K Q^T
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tA, make_sw128_desc(k_base + c * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(q_base + c * 16384 + k * 32, 16, 1024), idKK, (c | k) != 0);
        umma_commit(s_full);
      }
      __syncwarp();
      mbar_wait(p_full, t & 1);  // Pd^T in smem; S^T read
      tc_fence_after();
      if (elect_one()) {  // (b) dV += Pd^T dO ; dP^T = V dO^T
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tdV, make_sw128_desc(ps + kb * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(do_base + kb * 8192 + k * 2048, 16384, 1024), idKM, (t > 0) || ((kb | k) != 0));
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tA, make_sw128_desc(v_base + c * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(do_base + c * 16384 + k * 32, 16, 1024), idKK, (c | k) != 0);
        umma_commit(dp_full);
      }
      __syncwarp();
      mbar_wait(ds_full, t & 1);  // dS^T in smem; dP^T read
      tc_fence_after();
      if (elect_one()) {  // (c) dK += dS^T Q ; dQ = dS K
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            umma_bf16(tdK, make_sw128_desc(ps + kb * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(q_base + kb * 8192 + k * 2048, 16384, 1024), idKM, (t > 0) || ((kb | k) != 0));
            umma_bf16(tA, make_sw128_desc(ps + kb * 8192 + k * 2048, 16384, 1024),
                      make_sw128_desc(k_base + kb * 8192 + k * 2048, 16384, 1024), idMM, (kb | k) != 0);
          }
        umma_commit(dq_full);
        umma_commit(qdo_empty);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------- softmax backward (thread = key row r) ----------------
    const int r = (warp - 4) * 32 + lane;
    const int key = j * 128 + r;
    const uint32_t t_lane = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const float mk = a.mask ? a.mask[(int64_t)b * a.s + key] * 1.4426950408889634f : 0.f;
    uint8_t* ps_s = smem + Cfg::OFF_PS;
    float* nl_s = reinterpret_cast<float*>(smem + Cfg::OFF_LSE);   // -lse2 per query (in place)
    const float* del_s = reinterpret_cast<const float*>(smem + Cfg::OFF_DELTA);
    uint32_t* bits_s = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BITS);  // [q][4 words] as loaded
    uint32_t* kbt_s = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_KBT);    // [4 words][q] transposed
    const uint32_t* kb_row = kbt_s + (r >> 5) * 128;  // this thread's key word, all 128 queries
    const int bit = r & 31;
    const float scale_log2 = a.scale_log2, inv_keep = a.inv_keep;
    for (int t = 0; t < nt; ++t) {
      const int i = i0 + t;
      const bool diag = a.causal && (i == j);
      mbar_wait(qdo_full, t & 1);  // lse / delta / bits of this query tile in smem
      {
        // per-tile preamble (thread r = query r): -lse (fully masked rows -> -inf so P = 0) and the
        // keep-bit words transposed so a thread reads 4 queries of its key word per 16-B load
        const float l2 = nl_s[r];
        nl_s[r] = (l2 == -INFINITY) ? -INFINITY : -l2;
        if (a.dropout) {
          const uint4 w = *reinterpret_cast<const uint4*>(bits_s + r * 4);
          kbt_s[r] = w.x;
          kbt_s[128 + r] = w.y;
          kbt_s[256 + r] = w.z;
          kbt_s[384 + r] = w.w;
        }
        named_barrier_sync(1, 128);
      }
      mbar_wait(s_full, t & 1);
      tc_fence_after();
      // P (bf16, kept for dS) and Pd^T = keep ? P : 0 -> smem, 32 queries per TMEM load
      uint32_t pp[64];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t sv[32];
        tmem_ld_32x32b_x32(tA + t_lane + cc * 32, sv);
        tmem_ld_wait();
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {  // 8 queries per 16-B granule
          const int c = cc * 4 + c4;
          const float4 n0 = *reinterpret_cast<const float4*>(nl_s + c * 8);
          const float4 n1 = *reinterpret_cast<const float4*>(nl_s + c * 8 + 4);
          const float nl[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
          uint32_t kw[8];
          if (a.dropout) {
            const uint4 k0 = *reinterpret_cast<const uint4*>(kb_row + c * 8);
            const uint4 k1 = *reinterpret_cast<const uint4*>(kb_row + c * 8 + 4);
            kw[0] = k0.x; kw[1] = k0.y; kw[2] = k0.z; kw[3] = k0.w;
            kw[4] = k1.x; kw[5] = k1.y; kw[6] = k1.z; kw[7] = k1.w;
          }
          float pr[8], pk[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int qq = c * 8 + e;
            pr[e] = ex2_approx(fmaf(__uint_as_float(sv[qq & 31]), scale_log2, mk + nl[e]));
          }
          if (diag) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (r > c * 8 + e) pr[e] = 0.f;
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) pk[e] = (!a.dropout || ((kw[e] >> bit) & 1u)) ? pr[e] : 0.f;
          uint32_t pd[4];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            pp[(c * 8 + e) >> 1] = pack_bf16x2(pr[e], pr[e + 1]);
            pd[e >> 1] = pack_bf16x2(pk[e], pk[e + 1]);
          }
          *reinterpret_cast<uint4*>(ps_s + (c >> 3) * 16384 + sw128_offset(r, c & 7)) =
              make_uint4(pd[0], pd[1], pd[2], pd[3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      // dS^T = P * (keep ? dP/(1-p) : 0  - Delta)
      mbar_wait(dp_full, t & 1);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t sv[32];
        tmem_ld_32x32b_x32(tA + t_lane + cc * 32, sv);
        tmem_ld_wait();
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const int c = cc * 4 + c4;
          const float4 d0 = *reinterpret_cast<const float4*>(del_s + c * 8);
          const float4 d1 = *reinterpret_cast<const float4*>(del_s + c * 8 + 4);
          const float dl[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
          uint32_t kw[8];
          if (a.dropout) {
            const uint4 k0 = *reinterpret_cast<const uint4*>(kb_row + c * 8);
            const uint4 k1 = *reinterpret_cast<const uint4*>(kb_row + c * 8 + 4);
            kw[0] = k0.x; kw[1] = k0.y; kw[2] = k0.z; kw[3] = k0.w;
            kw[4] = k1.x; kw[5] = k1.y; kw[6] = k1.z; kw[7] = k1.w;
          }
          uint32_t dsw[4];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const float2 pf = unpack_bf16x2(pp[(c * 8 + e) >> 1]);
            float ds[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int qq = c * 8 + e + u;
              const bool kp = !a.dropout || ((kw[e + u] >> bit) & 1u);
              const float dp = kp ? __uint_as_float(sv[qq & 31]) * inv_keep : 0.f;
              ds[u] = (u ? pf.y : pf.x) * (dp - dl[e + u]);
            }
            dsw[e >> 1] = pack_bf16x2(ds[0], ds[1]);
          }
          *reinterpret_cast<uint4*>(ps_s + (c >> 3) * 16384 + sw128_offset(r, c & 7)) =
              make_uint4(dsw[0], dsw[1], dsw[2], dsw[3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      // drain dQ_i(j) (thread = query row r) as an fp32 partial
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
      float* dq = a.dq_part + ((int64_t)j * a.B * a.s + (int64_t)b * a.s + (int64_t)i * 128 + r) * a.H +
                  (int64_t)h * DH;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tA + t_lane + c * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 8; ++g)
          __stcg(reinterpret_cast<float4*>(dq + c * 32 + g * 4),
                 make_float4(__uint_as_float(o[g * 4]) * a.scale, __uint_as_float(o[g * 4 + 1]) * a.scale,
                             __uint_as_float(o[g * 4 + 2]) * a.scale, __uint_as_float(o[g * 4 + 3]) * a.scale));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_free);
    }
    // dK (scaled) and dV (1/(1-p)) rows of this key tile -> dqkv (bf16)
    bf16* dkrow = a.dqkv + ((int64_t)b * a.s + key) * a.ld + a.H + (int64_t)h * DH;
    bf16* dvrow = dkrow + a.H;
    const float sv_ = a.inv_keep;
#pragma unroll
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t kv[32], vv[32];
      tmem_ld_32x32b_x32(tdK + t_lane + c * 32, kv);
      tmem_ld_32x32b_x32(tdV + t_lane + c * 32, vv);
      tmem_ld_wait();
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint4 uk, uv;
        uk.x = pack_bf16x2(__uint_as_float(kv[g * 8 + 0]) * a.scale, __uint_as_float(kv[g * 8 + 1]) * a.scale);
        uk.y = pack_bf16x2(__uint_as_float(kv[g * 8 + 2]) * a.scale, __uint_as_float(kv[g * 8 + 3]) * a.scale);
        uk.z = pack_bf16x2(__uint_as_float(kv[g * 8 + 4]) * a.scale, __uint_as_float(kv[g * 8 + 5]) * a.scale);
        uk.w = pack_bf16x2(__uint_as_float(kv[g * 8 + 6]) * a.scale, __uint_as_float(kv[g * 8 + 7]) * a.scale);
        uv.x = pack_bf16x2(__uint_as_float(vv[g * 8 + 0]) * sv_, __uint_as_float(vv[g * 8 + 1]) * sv_);
        uv.y = pack_bf16x2(__uint_as_float(vv[g * 8 + 2]) * sv_, __uint_as_float(vv[g * 8 + 3]) * sv_);
        uv.z = pack_bf16x2(__uint_as_float(vv[g * 8 + 4]) * sv_, __uint_as_float(vv[g * 8 + 5]) * sv_);
        uv.w = pack_bf16x2(__uint_as_float(vv[g * 8 + 6]) * sv_, __uint_as_float(vv[g * 8 + 7]) * sv_);
        *reinterpret_cast<uint4*>(dkrow + c * 32 + g * 8) = uk;
        *reinterpret_cast<uint4*>(dvrow + c * 32 + g * 8) = uv;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, Cfg::TMEM_COLS);
  }
}

// ===========================================================================
// Pipelined backward (default).  CTA = (key tile j, head, sample), one CTA per SM, 512 threads:
//   warp 0      TMA producer: K_j, V_j once; per query tile i a stage {Q_i, dO_i, lse_i, Delta_i,
//               keep bits} (NQ stages: the next tile streams in while this one computes)
//   warp 1      MMA issuer:  S(t+1) = Q K^T into the other A buffer while tile t is in its
//               softmax passes; dV += Pd^T dO, dP = dO V^T; dK += dS^T Q, dQ = dS K (own region)
//   warp 2      TMEM allocator (512 columns)
//   warps 4-11  softmax backward, 8 warps: query row = TMEM lane (warp % 4), key half = warp / 4
//   warps 12-15 dQ drain (fp32 partial per key tile, summed in key-tile order by
//               smpk_flash_dq_reduce) overlapping the next tile, then the dK / dV epilogue
// TMEM: A0 [0,128), A1 [128,256) (S -> dP, NA = 2 buffers at dh = 64), dV, dK, dQ.
// ===========================================================================
constexpr int FB2_THREADS = 512;

// debug timeline (SMPK_FA_TRACE=1): per CTA 32 u64: [0] start [1] K/V landed (MMA warp), per tile t < 4:
// [2+t] S^T ready [6+t] P stored [10+t] dP^T ready [14+t] dS stored [18+t] dQ ready [22+t] dQ drained
// (elementwise warp 4 / drain warp 12, lane 0) [26] end [27] %smid
__device__ unsigned long long g_fb_trace[2048 * 64];
__device__ __forceinline__ unsigned long long gtime_b() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int DH>
struct FaBwd2Cfg {
  static constexpr int NA = DH == 64 ? 2 : 1;  // S^T / dP^T TMEM buffers
  static constexpr int NQ = DH == 64 ? 2 : 1;  // query-tile smem stages
  static constexpr int TILE = 128 * DH * 2;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + TILE;
  static constexpr int OFF_PDT = OFF_V + TILE;        // Pd^T (128 x 128 bf16)
  static constexpr int OFF_DST = OFF_PDT + 32768;     // dS^T
  static constexpr int OFF_STAGE = OFF_DST + 32768;   // NQ x {Q, dO, lse, Delta, bits}
  static constexpr int ST_Q = 0, ST_DO = TILE, ST_LSE = 2 * TILE, ST_DELTA = ST_LSE + 512, ST_BITS = ST_DELTA + 512;
  static constexpr int STAGE_BYTES = ST_BITS + 2048;
  static constexpr int OFF_KBT = OFF_STAGE + NQ * STAGE_BYTES;  // the key tile's additive mask (128 fp32)
  static constexpr int SG = DH == 64 ? 2 : 1;                   // dQ staging boxes [128 rows x 32 fp32]
  static constexpr int OFF_DQS = (OFF_KBT + 512 + 1023) / 1024 * 1024;
  static constexpr int OFF_BAR = OFF_DQS + SG * 16384;
  static constexpr int SMEM = 1024 + OFF_BAR + 256;
  static constexpr uint32_t COL_A = 0, COL_DV = NA * 128, COL_DK = COL_DV + DH, COL_DQ = COL_DK + DH;
  static_assert(COL_DQ + DH <= 512, "TMEM budget");
  static_assert(SMEM <= 232448, "smem budget");
};

template <int DH>
__global__ void __launch_bounds__(FB2_THREADS, 1)
    flash_bwd2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                      const __grid_constant__ CUtensorMap tmBits, const __grid_constant__ CUtensorMap tmDQ,
                      const FaBwdArgs a) {
  using Cfg = FaBwd2Cfg<DH>;
  constexpr int NA = Cfg::NA, NQ = Cfg::NQ;
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ array (not an integer round trip) keeps the shared
  // address space visible to the compiler: LDS / STS instead of generic LD / ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* qdo_full = bar + 1;   // [NQ]
  uint64_t* qdo_empty = bar + 3;  // [NQ]
  uint64_t* s_full = bar + 5;     // [NA]
  uint64_t* p_full = bar + 7;
  uint64_t* dp_full = bar + 8;
  uint64_t* ds_full = bar + 9;
  uint64_t* pdt_free = bar + 10;
  uint64_t* dst_free = bar + 11;
  uint64_t* dq_full = bar + 12;
  uint64_t* dq_free = bar + 13;
  uint64_t* kv_done = bar + 14;
  uint64_t* dqa_full = bar + 15;  // the earlier key tiles' dQ sum landed in the staging boxes
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);
  uint64_t* dst_drained = bar + 17;  // dh 128: the dQ drain is done with the dS^T buffer it borrowed

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_kt = a.s / 128;
  const int j = a.causal ? n_kt - 1 - (int)blockIdx.x : (int)blockIdx.x;  // key tile
  const int h = blockIdx.y, b = blockIdx.z;
  // query tile processed at step t: causal i = j + t; otherwise rotated, i = (j + t) mod n_kt, so the
  // key-tile CTAs of one (head, sample) work on different query tiles at every step and tile i's
  // dQ contributions arrive in step order (contribution number t; see the drain warps): the CTA
  // of contribution t waits for key tile j+1's CTA, which did its part one step earlier.  Causal
  // groups launch key tiles in descending order (blockIdx.x = n_kt-1-j), so that predecessor was
  // always launched first: no wait on a not-yet-resident block.
  const int nt = a.causal ? n_kt - j : n_kt;
  auto qtile = [&](int t) { return a.causal ? j + t : (j + t) % n_kt; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmDO);
    if (a.dropout) tma_prefetch_desc(&tmBits);
    mbar_init(kv_full, 1);
    for (int u = 0; u < NQ; ++u) {
      mbar_init(&qdo_full[u], 1);
      mbar_init(&qdo_empty[u], 1);
    }
    for (int u = 0; u < NA; ++u) mbar_init(&s_full[u], 1);
    mbar_init(p_full, 8);  // one arrive per softmax warp
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 8);
    mbar_init(pdt_free, 1);
    mbar_init(dst_free, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);  // one arrive per drain warp
    mbar_init(kv_done, 1);
    mbar_init(dqa_full, 1);
    mbar_init(dst_drained, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  const int64_t bh_row = ((int64_t)b * a.nh + h) * a.s;
  const int cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  unsigned long long* trc = (a.trace && cta_lin < 2048) ? g_fb_trace + cta_lin * 64 : nullptr;
  if (trc && threadIdx.x == 0) {
    trc[0] = gtime_b();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    trc[27] = smid;
  }
#define FB_TR(slot)                                      \
  do {                                                   \
    if (trc && lane == 0 && t < 4) trc[(slot) + t] = gtime_b(); \
  } while (0)

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_arrive_expect_tx(kv_full, 2 * Cfg::TILE);
#pragma unroll
      for (int c = 0; c < DH / 64; ++c) {
        tma_load_4d(smem + Cfg::OFF_K + c * 16384, &tmK, kv_full, c * 64, j * 128, h, b);
        tma_load_4d(smem + Cfg::OFF_V + c * 16384, &tmV, kv_full, c * 64, j * 128, h, b);
      }
      for (int t = 0; t < nt; ++t) {
        const int i = qtile(t), u = t % NQ;
        if (t >= NQ) mbar_wait(&qdo_empty[u], ((t / NQ) - 1) & 1);
        uint8_t* stg = smem + Cfg::OFF_STAGE + u * Cfg::STAGE_BYTES;
        mbar_arrive_expect_tx(&qdo_full[u], 2 * Cfg::TILE + 1024 + (a.dropout ? 2048 : 0));
        const int64_t off = bh_row + (int64_t)i * 128;
#pragma unroll
        for (int c = 0; c < DH / 64; ++c) {
          tma_load_4d(stg + Cfg::ST_Q + c * 16384, &tmQ, &qdo_full[u], c * 64, i * 128, h, b);
          tma_load_4d(stg + Cfg::ST_DO + c * 16384, &tmDO, &qdo_full[u], c * 64, i * 128, h, b);
        }
        bulk_load(stg + Cfg::ST_LSE, a.lse + off, 512, &qdo_full[u]);
        bulk_load(stg + Cfg::ST_DELTA, a.delta + off, 512, &qdo_full[u]);
        if (a.dropout) tma_load_4d(stg + Cfg::ST_BITS, &tmBits, &qdo_full[u], j * 4, (int)off, 0, 0);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp; one elected lane issues) ----------------
    // Query rows on the TMEM lanes: S = Q K^T and dP = dO V^T (M = queries); P / dS live in smem
    // as [query rows x keys] (K-major for dQ = dS K, and the MN-major A operand of
    // dV += P^T dO / dK += dS^T Q, M = keys).
    const uint32_t idQK = make_idesc_bf16(128, 128, false, false);  // S, dP
    const uint32_t idTM = make_idesc_bf16(128, DH, true, true);     // dV, dK: A = P^T / dS^T (MN-major)
    const uint32_t idKM = make_idesc_bf16(128, DH, false, true);    // dQ: A = dS (K-major), B = K (MN-major)
    const uint32_t k_base = smem_u32(smem + Cfg::OFF_K), v_base = smem_u32(smem + Cfg::OFF_V);
    const uint32_t pdt = smem_u32(smem + Cfg::OFF_PDT), dst = smem_u32(smem + Cfg::OFF_DST);
    const uint32_t tdV = tmem + Cfg::COL_DV, tdK = tmem + Cfg::COL_DK, tdQ = tmem + Cfg::COL_DQ;
    auto stage_base = [&](int t) { return smem_u32(smem + Cfg::OFF_STAGE + (t % NQ) * Cfg::STAGE_BYTES); };
    // TMEM: with NA == 2 (dh 64) S(t) always lands in A0 and dP(t) in A1, so the next tile's S is
    // computed during this tile's dS pass and the next dP during the next P pass -- neither pass
    // waits on an MMA.  With NA == 1 (dh 128: no room for a second 128-column buffer) S and dP
    // share A.  In both, dK(t) is issued before waiting for the previous dQ drain and the Q / dO
    // stage is released right after it, so the next tile's loads overlap that drain.
    auto issue_s = [&](int t) {  // S(t) = Q_t K^T -> A0
      mbar_wait(&qdo_full[t % NQ], (t / NQ) & 1);
      tc_fence_after();
      const uint32_t qb = stage_base(t) + Cfg::ST_Q;
      if (elect_one()) {
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem, make_sw128_desc(qb + c * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(k_base + c * 16384 + k * 32, 16, 1024), idQK, (c | k) != 0);
        umma_commit(&s_full[0]);
      }
      __syncwarp();
    };
    auto issue_dp = [&](int t) {  // dP(t) = dO_t V^T -> A[NA - 1] (stage t already waited by issue_s)
      const uint32_t dob = stage_base(t) + Cfg::ST_DO;
      if (elect_one()) {
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem + (NA - 1) * 128, make_sw128_desc(dob + c * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(v_base + c * 16384 + k * 32, 16, 1024), idQK, (c | k) != 0);
        umma_commit(dp_full);
      }
      __syncwarp();
    };
    mbar_wait(kv_full, 0);
    if (trc && lane == 0) trc[1] = gtime_b();
    if (nt > 0) {
      issue_s(0);
      if (NA == 2) issue_dp(0);
    }
    for (int t = 0; t < nt; ++t) {
      const uint32_t dob = stage_base(t) + Cfg::ST_DO, qb = stage_base(t) + Cfg::ST_Q;
      mbar_wait(p_full, t & 1);  // Pd(t) in smem; S(t) read
      tc_fence_after();
      if (elect_one()) {  // dV += Pd^T dO
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_bf16(tdV, make_sw128_desc(pdt + k * 2048, 16384, 1024), make_sw128_desc(dob + k * 2048, 16384, 1024),
                    idTM, (t > 0) || (k != 0));
        umma_commit(pdt_free);
      }
      __syncwarp();
      if (NA == 1) issue_dp(t);                // A is free once S(t) was read
      else if (t + 1 < nt) issue_s(t + 1);     // A0 is free: the next scores during this dS pass
      mbar_wait(ds_full, t & 1);  // dS(t) in smem; dP(t) read
      tc_fence_after();
      if (elect_one()) {  // dK += dS^T Q, then the Q / dO stage can be refilled
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_bf16(tdK, make_sw128_desc(dst + k * 2048, 16384, 1024), make_sw128_desc(qb + k * 2048, 16384, 1024),
                    idTM, (t > 0) || (k != 0));
        umma_commit(&qdo_empty[t % NQ]);
      }
      __syncwarp();
      if (NA == 2 && t + 1 < nt) issue_dp(t + 1);  // A1 is free once dP(t) was read
      if (t > 0) mbar_wait(dq_free, (t - 1) & 1);  // dQ(t-1) drained
      tc_fence_after();
      if (elect_one()) {  // dQ = dS K
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tdQ, make_sw128_desc(dst + kb * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(k_base + kb * 8192 + k * 2048, 16384, 1024), idKM, (kb | k) != 0);
        umma_commit(dq_full);
        umma_commit(dst_free);
        if (t == nt - 1) umma_commit(kv_done);
      }
      __syncwarp();
      if (NA == 1 && t + 1 < nt) issue_s(t + 1);  // A is free once dP(t) was read
    }
  } else if (warp >= 4 && warp < 12) {
    // ---------------- softmax backward: query row qr = TMEM lane, 64 keys per warp ----------------
    // per-query lse / Delta are per-thread scalars and the keep bits of (query, 64 keys) are two
    // words of the thread's own row, so the shared-memory traffic per element is the 2-byte P / dS
    // store only (the MIO queue was the limiter with key rows on the lanes)
    const int e = warp - 4;
    const int lq = e & 3, qh = e >> 2;
    const int qr = lq * 32 + lane;
    const uint32_t t_lane = static_cast<uint32_t>(lq * 32) << 16;
    uint8_t* pd_s = smem + Cfg::OFF_PDT + qh * 16384;  // this warp's 64-key chunk
    uint8_t* ds_s = smem + Cfg::OFF_DST + qh * 16384;
    float* mk_s = reinterpret_cast<float*>(smem + Cfg::OFF_KBT);  // additive mask (log2 domain) of the keys
    const int tid = threadIdx.x - 128;  // 0..255
    if (a.mask) {
      if (tid < 128) mk_s[tid] = a.mask[(int64_t)b * a.s + j * 128 + tid] * 1.4426950408889634f;
      named_barrier_sync(1, 256);
    }
    const float scale_log2 = a.scale_log2, inv_keep = a.inv_keep;
    for (int t = 0; t < nt; ++t) {
      const int i = qtile(t);
      const bool diag = a.causal && (i == j);
      const uint8_t* stg = smem + Cfg::OFF_STAGE + (t % NQ) * Cfg::STAGE_BYTES;
      mbar_wait(&qdo_full[t % NQ], (t / NQ) & 1);
      const float nls = -reinterpret_cast<const float*>(stg + Cfg::ST_LSE)[qr];  // +inf lse: masked row
      const float dlt = reinterpret_cast<const float*>(stg + Cfg::ST_DELTA)[qr];
      uint32_t kw0 = 0xffffffffu, kw1 = 0xffffffffu;
      if (a.dropout) {
        const uint2 w = *reinterpret_cast<const uint2*>(stg + Cfg::ST_BITS + qr * 16 + qh * 8);
        kw0 = w.x;
        kw1 = w.y;
      }
      mbar_wait(&s_full[0], t & 1);
      if (e == 0) FB_TR(2);
      tc_fence_after();
      const uint32_t tA = tmem + t_lane + qh * 64;               // S(t)
      const uint32_t tP = tmem + (NA - 1) * 128 + t_lane + qh * 64;  // dP(t)
      // ---- P pass: P (bf16, kept for dS) and Pd = keep ? P : 0 -> smem
      uint32_t pp[32];
      uint32_t sv[64];
      tmem_ld_32x32b_x32(tA, *reinterpret_cast<uint32_t(*)[32]>(sv));
      tmem_ld_32x32b_x32(tA + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
      tmem_ld_wait();
      if (e == 0) FB_TR(32);
      if (t > 0) mbar_wait(pdt_free, (t - 1) & 1);  // dV(t-1) has read Pd
      if (e == 0) FB_TR(36);
      // paired fp32 math (FFMA2) and packed keep masks: the pass is issue-bound
      const float2 sc2 = make_float2(scale_log2, scale_log2), nls2 = make_float2(nls, nls);
      uint32_t ksh[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // 8 keys per 16-B granule
        if ((c & 3) == 0) keep_shifts(c < 4 ? kw0 : kw1, ksh);
        float pr[8];
        if (a.mask) {
          const float4 m0 = *reinterpret_cast<const float4*>(mk_s + qh * 64 + c * 8);
          const float4 m1 = *reinterpret_cast<const float4*>(mk_s + qh * 64 + c * 8 + 4);
          const float mm[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
          for (int u = 0; u < 8; u += 2) {
            const float2 y = __ffma2_rn(make_float2(__uint_as_float(sv[c * 8 + u]), __uint_as_float(sv[c * 8 + u + 1])),
                                        sc2, __fadd2_rn(make_float2(mm[u], mm[u + 1]), nls2));
            pr[u] = ex2_approx(y.x);
            pr[u + 1] = ex2_approx(y.y);
          }
        } else {
#pragma unroll
          for (int u = 0; u < 8; u += 2) {
            const float2 y = __ffma2_rn(make_float2(__uint_as_float(sv[c * 8 + u]), __uint_as_float(sv[c * 8 + u + 1])),
                                        sc2, nls2);
            pr[u] = ex2_approx(y.x);
            pr[u + 1] = ex2_approx(y.y);
          }
        }
        if (diag) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (qh * 64 + c * 8 + u > qr) pr[u] = 0.f;  // key after query
        }
        uint32_t pd[4];
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          const uint32_t p2 = pack_bf16x2(pr[u], pr[u + 1]);
          pp[(c * 8 + u) >> 1] = p2;
          pd[u >> 1] = p2 & keep_pair_mask(ksh, c & 3, u);
        }
        *reinterpret_cast<uint4*>(pd_s + sw128_offset(qr, c)) = make_uint4(pd[0], pd[1], pd[2], pd[3]);
      }
      if (e == 0) FB_TR(40);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (e == 0) FB_TR(6);
      // ---- dS pass: dS = P * (keep ? dP/(1-p) : 0  - Delta)
      mbar_wait(dp_full, t & 1);
      if (e == 0) FB_TR(10);
      tc_fence_after();
      tmem_ld_32x32b_x32(tP, *reinterpret_cast<uint32_t(*)[32]>(sv));
      tmem_ld_32x32b_x32(tP + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
      tmem_ld_wait();
      if (t > 0) mbar_wait(dst_free, (t - 1) & 1);  // dK / dQ(t-1) have read dS
      if (DH == 128 && t > 0) mbar_wait(dst_drained, (t - 1) & 1);  // the dQ(t-1) drain returned it
      const float2 ik2 = make_float2(inv_keep, inv_keep), nd2 = make_float2(-dlt, -dlt);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t w = c < 4 ? kw0 : kw1;
        const int sh = (c & 3) * 8;
        uint32_t dsw[4];
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          const float2 pf = unpack_bf16x2(pp[(c * 8 + u) >> 1]);
          float2 d = __ffma2_rn(make_float2(__uint_as_float(sv[c * 8 + u]), __uint_as_float(sv[c * 8 + u + 1])), ik2,
                                nd2);  // dP/(1-p) - Delta
          if (!((w >> (sh + u)) & 1u)) d.x = -dlt;
          if (!((w >> (sh + u + 1)) & 1u)) d.y = -dlt;
          const float2 r = __fmul2_rn(pf, d);
          dsw[u >> 1] = pack_bf16x2(r.x, r.y);
        }
        *reinterpret_cast<uint4*>(ds_s + sw128_offset(qr, c)) = make_uint4(dsw[0], dsw[1], dsw[2], dsw[3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      if (e == 0) FB_TR(14);
    }
    // dK (scaled; warps 4-7) and dV (1/(1-p); warps 8-11) rows of this key tile -> dqkv (bf16),
    // written while the drain warps finish the last dQ tile
    if (nt > 0) {
      mbar_wait(kv_done, 0);
      tc_fence_after();
    }
    {
      const int key = j * 128 + qr;  // key row = TMEM lane of the dK / dV accumulators
      bf16* orow = a.dqkv + ((int64_t)b * a.s + key) * a.ld + (qh ? 2 * a.H : a.H) + (int64_t)h * DH;
      const float sc = qh ? a.inv_keep : a.scale;
      const uint32_t col = qh ? Cfg::COL_DV : Cfg::COL_DK;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t kv[32];
        if (nt > 0) {
          tmem_ld_32x32b_x32(tmem + col + t_lane + c * 32, kv);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) kv[q] = 0u;
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint4 u;
          u.x = pack_bf16x2(__uint_as_float(kv[g * 8 + 0]) * sc, __uint_as_float(kv[g * 8 + 1]) * sc);
          u.y = pack_bf16x2(__uint_as_float(kv[g * 8 + 2]) * sc, __uint_as_float(kv[g * 8 + 3]) * sc);
          u.z = pack_bf16x2(__uint_as_float(kv[g * 8 + 4]) * sc, __uint_as_float(kv[g * 8 + 5]) * sc);
          u.w = pack_bf16x2(__uint_as_float(kv[g * 8 + 6]) * sc, __uint_as_float(kv[g * 8 + 7]) * sc);
          *reinterpret_cast<uint4*>(orow + c * 32 + g * 8) = u;
        }
      }
    }
  } else if (warp >= 12) {
    // ---------------- dQ drain (query row = TMEM lane), then the dK / dV epilogue ----------------
    // dQ of query tile i is the sum over key tiles j of dS_ij K_j.  The key-tile CTAs add their
    // terms into an fp32 accumulator in ascending j order (bit-deterministic): j = 0 TMA-stores,
    // later ones TMA reduce-add (the add happens in L2, off the SM's load/store pipe), each after
    // the previous contributor released the tile's counter; the last contributor instead loads
    // the sum of the others, adds its own term in registers and writes bf16 dQ into dqkv.
    const int lq = warp & 3;
    const int rr = lq * 32 + lane;
    const uint32_t t_lane = static_cast<uint32_t>(lq * 32) << 16;
    const bool issuer = (warp == 12 && lane == 0);
    uint8_t* dqs = smem + Cfg::OFF_DQS;
    uint32_t dqa_phase = 0;
    int* cnt_base = a.dq_cnt + ((int64_t)b * a.nh + h) * n_kt;
    for (int t = 0; t < nt; ++t) {
      const int i = qtile(t);
      // this CTA is contribution number t of query tile i's dQ (causal: key tiles i, i-1, ..., 0;
      // otherwise j = i, i-1, ... mod n_kt): wait until t earlier contributions are complete
      const int ncontrib = a.causal ? i + 1 : n_kt;
      const bool firstc = (t == 0), lastc = (t == ncontrib - 1);
      int* cnt = cnt_base + i;
      const int row0 = b * a.s + i * 128;
      mbar_wait(dq_full, t & 1);
      if (warp == 12) FB_TR(18);
      if (DH == 128 && lastc && issuer) mbar_arrive(dst_drained);  // not borrowed: phases stay in step
      tc_fence_after();
      bool my_turn = firstc;  // (issuer) the previous contributors are done with this tile
#pragma unroll 1
      for (int hf = 0; hf < DH / 64; ++hf) {
        uint32_t o[64];
        tmem_ld_32x32b_x32(tmem + Cfg::COL_DQ + t_lane + hf * 64, *reinterpret_cast<uint32_t(*)[32]>(o));
        tmem_ld_32x32b_x32(tmem + Cfg::COL_DQ + t_lane + hf * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(o + 32));
        tmem_ld_wait();
        if (hf == DH / 64 - 1) {  // dQ(t) is in registers: the next dQ MMA may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dq_free);
        }
        float* v = reinterpret_cast<float*>(o);
#pragma unroll
        for (int q = 0; q < 64; ++q) v[q] = __uint_as_float(o[q]) * a.scale;
        if (DH == 128 && !lastc) {
          // dh 128 has room for one 16 KB staging box only; the dS^T buffer (32 KB) is idle from the
          // end of the dQ(t) MMA until the next dS pass, so chunks 1 and 2 of the four 32-column
          // chunks are staged there -- only after this tile's turn came, so the borrow is short --
          // and it is handed back (dst_drained) once the TMA engine has read them
          uint8_t* dsb = smem + Cfg::OFF_DST;
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            const int cidx = hf * 2 + g;  // 32-column chunk 0..3
            uint8_t* boxb = (cidx == 1 || cidx == 2) ? dsb + (cidx - 1) * 16384 : dqs;
            uint8_t* box = boxb + rr * 128;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float* src = v + g * 32 + q * 4;
              *reinterpret_cast<float4*>(box + ((q ^ (rr & 7)) << 4)) = make_float4(src[0], src[1], src[2], src[3]);
            }
            fence_proxy_async_smem();
            named_barrier_sync(3, 128);
            if (issuer) {
              if (!my_turn) {
                while (ld_acquire_gpu(cnt) != t) __nanosleep(32);
                fence_proxy_async_global();
                my_turn = true;
              }
              const int c0 = h * DH + cidx * 32;
              if (firstc)
                tma_store_2d(&tmDQ, boxb, c0, row0);
              else
                tma_reduce_add_2d(&tmDQ, boxb, c0, row0);
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
              if (cidx == 2) {  // chunks 0-2 read: the dS^T buffer goes back, the box is reusable
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                mbar_arrive(dst_drained);
              }
              if (cidx == 3) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            named_barrier_sync(3, 128);
          }
        } else if (!lastc) {
#pragma unroll
          for (int g0 = 0; g0 < 2; g0 += Cfg::SG) {
#pragma unroll
            for (int gg = 0; gg < Cfg::SG; ++gg) {
              uint8_t* box = dqs + gg * 16384 + rr * 128;
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float* src = v + (g0 + gg) * 32 + q * 4;
                *reinterpret_cast<float4*>(box + ((q ^ (rr & 7)) << 4)) = make_float4(src[0], src[1], src[2], src[3]);
              }
            }
            fence_proxy_async_smem();
            named_barrier_sync(3, 128);
            if (issuer) {
              if (!my_turn) {
                while (ld_acquire_gpu(cnt) != t) __nanosleep(32);
                fence_proxy_async_global();
                my_turn = true;
              }
#pragma unroll
              for (int gg = 0; gg < Cfg::SG; ++gg) {
                const int c0 = h * DH + hf * 64 + (g0 + gg) * 32;
                if (firstc)
                  tma_store_2d(&tmDQ, dqs + gg * 16384, c0, row0);
                else
                  tma_reduce_add_2d(&tmDQ, dqs + gg * 16384, c0, row0);
              }
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging reusable
            }
            named_barrier_sync(3, 128);
          }
        } else {
          if (!firstc) {  // add the earlier key tiles' sum
#pragma unroll
            for (int g0 = 0; g0 < 2; g0 += Cfg::SG) {
              if (issuer) {
                if (!my_turn) {
                  while (ld_acquire_gpu(cnt) != t) __nanosleep(32);
                  fence_proxy_async_global();
                  my_turn = true;
                }
                mbar_arrive_expect_tx(dqa_full, Cfg::SG * 16384);
#pragma unroll
                for (int gg = 0; gg < Cfg::SG; ++gg)
                  tma_load_4d(dqs + gg * 16384, &tmDQ, dqa_full, h * DH + hf * 64 + (g0 + gg) * 32, row0, 0, 0);
              }
              mbar_wait(dqa_full, dqa_phase);
              dqa_phase ^= 1;
#pragma unroll
              for (int gg = 0; gg < Cfg::SG; ++gg) {
                const uint8_t* box = dqs + gg * 16384 + rr * 128;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                  const float4 s4 = *reinterpret_cast<const float4*>(box + ((q ^ (rr & 7)) << 4));
                  float* dv = v + (g0 + gg) * 32 + q * 4;
                  dv[0] = s4.x + dv[0];
                  dv[1] = s4.y + dv[1];
                  dv[2] = s4.z + dv[2];
                  dv[3] = s4.w + dv[3];
                }
              }
              named_barrier_sync(3, 128);  // staging read by every drain thread
            }
          }
          bf16* dqrow = a.dqkv + (int64_t)(row0 + rr) * a.ld + (int64_t)h * DH + hf * 64;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            uint4 u;
            u.x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
            u.y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
            u.z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
            u.w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
            *reinterpret_cast<uint4*>(dqrow + q * 8) = u;
          }
        }
      }
      if (issuer) {
        if (!lastc) {  // release the tile to the next key tile: our adds are complete in L2
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          fence_proxy_async_global();
          __threadfence();
          st_release_gpu(cnt, t + 1);
        } else if (!firstc) {
          *cnt = 0;  // every contributor is done: reset for the next launch / graph replay
        }
      }
      if (warp == 12) FB_TR(22);
    }
    if (trc && threadIdx.x == 384) trc[26] = gtime_b();
  }
#undef FB_TR
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Delta[b, h, q] = sum_d dO[b*s+q, h*dh+d] * O[b*s+q, h*dh+d]
// 8 lanes per (row, head): each lane loads 16 B of O and dO per 64 columns (coalesced 128-byte
// segments, every load of the head issued up front), then a 3-step xor-shuffle sum.
__global__ void __launch_bounds__(256) flash_delta_kernel(const bf16* __restrict__ o, int64_t ld_o,
                                                          const bf16* __restrict__ dout, int64_t ld_do, int B,
                                                          int nh, int s, int dh, float* __restrict__ delta,
                                                          int* __restrict__ cnt, int n_cnt) {
  pdl_trigger();
  pdl_wait();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (cnt && t < n_cnt) cnt[t] = 0;  // the backward's per-query-tile dQ turn counters
  const int64_t idx = t >> 3;
  const int sub = (int)(t & 7);
  const int64_t total = (int64_t)B * s * nh;
  const bool valid = idx < total;  // no early exit: the whole warp takes part in the shuffles
  const int h = valid ? (int)(idx % nh) : 0;
  const int64_t row = valid ? idx / nh : 0;
  float acc = 0.f;
  if (valid) {
    const bf16* op = o + row * ld_o + (int64_t)h * dh;
    const bf16* dp = dout + row * ld_do + (int64_t)h * dh;
#pragma unroll 2
    for (int d = sub * 8; d < dh; d += 64) {
      const uint4 a = *reinterpret_cast<const uint4*>(op + d);
      const uint4 c = *reinterpret_cast<const uint4*>(dp + d);
      const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 fa = unpack_bf16x2(wa[k]), fc = unpack_bf16x2(wc[k]);
        acc += fa.x * fc.x + fa.y * fc.y;
      }
    }
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  if (valid && sub == 0) {
    const int64_t b = row / s, q = row % s;
    delta[(b * nh + h) * s + q] = acc;
  }
}

// dQ[row, col] = sum over key tiles j (j <= row's query tile if causal) of dq_part[j][row][col]
__global__ void flash_dq_reduce_kernel(const float* __restrict__ part, int n_kt, int64_t rows, int64_t H, int s,
                                       int causal, bf16* __restrict__ dq, int64_t ld) {
  const int64_t idx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (idx >= rows * H) return;
  const int64_t row = idx / H, col = idx % H;
  const int qt = (int)((row % s) / 128);
  const int jmax = causal ? qt : n_kt - 1;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int jj = 0; jj <= jmax; ++jj) {
    float4 v = *reinterpret_cast<const float4*>(part + ((int64_t)jj * rows + row) * H + col);
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  uint2 u;
  u.x = pack_bf16x2(acc.x, acc.y);
  u.y = pack_bf16x2(acc.z, acc.w);
  *reinterpret_cast<uint2*>(dq + row * ld + col) = u;
}

}  // namespace smpk

using namespace smpk;

static bool bwd_v1() {
  static int v1 = -1;
  if (v1 < 0) {
    const char* e = getenv("SMPK_FA_BWD_V1");
    v1 = (e && e[0] == '1') ? 1 : 0;
  }
  return v1 == 1;
}

// default kernel: fp32 dQ accumulator [B*s, H] + Delta [B, nh, s] + turn counters [B, nh, s/128];
// SMPK_FA_BWD_V1=1 (A/B reference): one fp32 dQ partial per key tile + Delta
extern "C" int64_t smpk_flash_attn_bwd_workspace(int B, int nh, int s, int dh) {
  const int64_t n_kt = s / 128;
  const int64_t acc = (bwd_v1() ? n_kt : 1) * (int64_t)B * s * nh * dh * 4;
  return acc + (int64_t)B * nh * s * 4 + (int64_t)B * nh * n_kt * 4;
}

extern "C" int smpk_flash_attn_bwd(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* dout,
                                   int64_t ld_dout, const float* lse, int B, int nh, int s, int dh, void* dqkv,
                                   const float* mask_add, float scale, int causal, float p_drop,
                                   const uint32_t* keep_bits, void* workspace, int64_t workspace_bytes, void* stream) {
  SMPK_REQUIRE(dh == 64 || dh == 128, SMPK_ERR_UNSUPPORTED, "smpk_flash_attn_bwd: head dim %d (64 or 128)", dh);
  SMPK_REQUIRE(s % 128 == 0 && s > 0, SMPK_ERR_UNSUPPORTED, "smpk_flash_attn_bwd: seq %d must be a multiple of 128",
               s);
  SMPK_REQUIRE(qkv && out && dout && lse && dqkv, SMPK_ERR_BAD_ARG, "smpk_flash_attn_bwd: null argument");
  SMPK_REQUIRE(p_drop == 0.f || keep_bits, SMPK_ERR_BAD_ARG, "smpk_flash_attn_bwd: dropout needs keep bits");
  SMPK_REQUIRE(ld % 8 == 0 && ld_out % 8 == 0 && ld_dout % 8 == 0, SMPK_ERR_BAD_ARG,
               "smpk_flash_attn_bwd: leading dims must be multiples of 8");
  const int64_t need = smpk_flash_attn_bwd_workspace(B, nh, s, dh);
  SMPK_REQUIRE(workspace && workspace_bytes >= need, SMPK_ERR_BAD_ARG, "smpk_flash_attn_bwd: workspace too small");
  const bool v1 = bwd_v1();
  const int64_t H = (int64_t)nh * dh;
  const int n_kt = s / 128;
  float* dq_part = reinterpret_cast<float*>(workspace);
  float* delta = dq_part + (v1 ? (int64_t)n_kt : 1) * B * s * H;
  int* cnt = reinterpret_cast<int*>(delta + (int64_t)B * nh * s);
  const int n_cnt = B * nh * n_kt;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  {
    const int64_t total = (int64_t)B * s * nh;
    launch_pdl(flash_delta_kernel, dim3((unsigned)((total * 8 + 255) / 256)), dim3(256), 0, st,
               reinterpret_cast<const bf16*>(out), ld_out, reinterpret_cast<const bf16*>(dout), ld_dout, B, nh, s,
               dh, delta, cnt, n_cnt);
    int rc = check_launch("smpk_flash_attn_bwd(delta)");
    if (rc) return rc;
  }
  const bf16* base = reinterpret_cast<const bf16*>(qkv);
  CUtensorMap tq, tk, tv, tdo;
  int rc = make_tma_4d(&tq, base, dh, s, ld, nh, dh, B, (int64_t)s * ld, 64, 128, "Q");
  if (!rc) rc = make_tma_4d(&tk, base + H, dh, s, ld, nh, dh, B, (int64_t)s * ld, 64, 128, "K");
  if (!rc) rc = make_tma_4d(&tv, base + 2 * H, dh, s, ld, nh, dh, B, (int64_t)s * ld, 64, 128, "V");
  if (!rc) rc = make_tma_4d(&tdo, dout, dh, s, ld_dout, nh, dh, B, (int64_t)s * ld_dout, 64, 128, "dO");
  CUtensorMap tbits;
  memset(&tbits, 0, sizeof(tbits));
  if (!rc && p_drop > 0.f)
    rc = make_tma_4d_b32(&tbits, keep_bits, s / 32, (int64_t)B * nh * s, s / 32, 4, 128, "keep bits");
  if (rc) return rc;
  FaBwdArgs a;
  a.B = B;
  a.nh = nh;
  a.s = s;
  a.lse = lse;
  a.delta = delta;
  a.mask = mask_add;
  a.scale = scale;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.causal = causal;
  a.dropout = p_drop > 0.f ? 1 : 0;
  a.inv_keep = p_drop > 0.f ? 1.f / (1.f - p_drop) : 1.f;
  a.dqkv = reinterpret_cast<bf16*>(dqkv);
  a.ld = ld;
  a.H = H;
  a.dq_part = dq_part;
  a.dq_cnt = cnt;
  static int trace_env = -1;
  if (trace_env < 0) {
    const char* e = getenv("SMPK_FA_TRACE");
    trace_env = e ? atoi(e) : 0;
  }
  a.trace = trace_env;
  dim3 grid(n_kt, nh, B);
  if (!v1) {
    CUtensorMap tdq;
    rc = make_tma_4d_f32sw(&tdq, dq_part, H, (int64_t)B * s, H, 32, 128, "dQ accumulator");
    if (rc) return rc;
    if (dh == 64) {
      static unsigned long long once = 0;
      smem_attr_once(flash_bwd2_kernel<64>, FaBwd2Cfg<64>::SMEM, once);
      launch_pdl(flash_bwd2_kernel<64>, grid, FB2_THREADS, FaBwd2Cfg<64>::SMEM, st, tq, tk, tv, tdo, tbits, tdq, a);
    } else {
      static unsigned long long once = 0;
      smem_attr_once(flash_bwd2_kernel<128>, FaBwd2Cfg<128>::SMEM, once);
      launch_pdl(flash_bwd2_kernel<128>, grid, FB2_THREADS, FaBwd2Cfg<128>::SMEM, st, tq, tk, tv, tdo, tbits, tdq, a);
    }
    return check_launch("smpk_flash_attn_bwd");
  }
  if (dh == 64) {
    static unsigned long long once = 0;
    smem_attr_once(flash_bwd_kernel<64>, FaBwdCfg<64>::SMEM, once);
    flash_bwd_kernel<64><<<grid, FB_THREADS, FaBwdCfg<64>::SMEM, st>>>(tq, tk, tv, tdo, tbits, a);
  } else {
    static unsigned long long once = 0;
    smem_attr_once(flash_bwd_kernel<128>, FaBwdCfg<128>::SMEM, once);
    flash_bwd_kernel<128><<<grid, FB_THREADS, FaBwdCfg<128>::SMEM, st>>>(tq, tk, tv, tdo, tbits, a);
  }
  rc = check_launch("smpk_flash_attn_bwd");
  if (rc) return rc;
  const int64_t n4 = (int64_t)B * s * H / 4;
  flash_dq_reduce_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(dq_part, n_kt, (int64_t)B * s, H, s, causal,
                                                                      reinterpret_cast<bf16*>(dqkv), ld);
  return check_launch("smpk_flash_attn_bwd(dq reduce)");
}

extern "C" int smpk_debug_fb_trace(void* host_out, int n_cta) {
  if (n_cta > 2048) n_cta = 2048;
  cudaError_t e = cudaMemcpyFromSymbol(host_out, smpk::g_fb_trace, (size_t)n_cta * 64 * 8);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_debug_fb_trace: %s", cudaGetErrorString(e));
  return SMPK_OK;
}

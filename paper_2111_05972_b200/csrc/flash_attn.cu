// flash_attn.cu — fused attention forward on tcgen05/TMEM/TMA (sm_100a).
//
// The attention core of dist_attention_forward for one TP rank's
// local heads: softmax(Q K^T / sqrt(dh) + mask [+ causal]) -> dropout -> . V, without
// materialising the [s, s] score / probability matrices in HBM.
//
// CTA = (128-row query tile, local head, sample); 256 threads:
//   warp 0   TMA producer: Q once, K/V tiles through a 2-stage ring
//   warp 1   MMA issuer:   S = Q K^T (M=128,N=128) into TMEM; O += P V (M=128,N=dh)
//   warp 2   TMEM allocator (256 columns: S 128 + O dh)
//   warps 4-7 softmax: thread = query row (TMEM lane); online max / sum in the exp2
//            domain, O rescaled in TMEM when the running max grows, dropout from the
//            Philox stream of oracle/philox.py, P written to smem as the bf16 K-major
//            A operand of the P.V MMA; final O / l and log-sum-exp stored.
// Two CTAs share an SM (TMEM 2 x 256 columns), so one CTA's softmax overlaps the
// other's tensor-core work.
#include "smpk_common.cuh"

namespace smpk {

constexpr int FA_THREADS = 256;
constexpr int FA_BQ = 128;
constexpr int FA_BK = 128;

struct FaFwdArgs {
  int B, nh, s;
  bf16* out;
  int64_t ld_out;
  float* lse;         // [B, nh, s] log2-domain log-sum-exp of the scaled+masked scores
  const float* mask;  // [B, s] additive, may be null
  float scale_log2;   // log2(e) / sqrt(dh)
  int causal;
  float p, inv_keep;
  uint32_t thresh;
  uint64_t seed;
  uint32_t layer;
  int64_t sample_offset;
  int head_offset, nh_global;
};

template <int DH>
struct FaFwdCfg {
  static constexpr int Q_BYTES = FA_BQ * DH * 2;
  static constexpr int K_BYTES = FA_BK * DH * 2;
  static constexpr int V_BYTES = FA_BK * DH * 2;
  static constexpr int P_BYTES = FA_BQ * FA_BK * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + 2 * K_BYTES;
  static constexpr int OFF_P = OFF_V + 2 * V_BYTES;
  static constexpr int OFF_BAR = OFF_P + P_BYTES;
  static constexpr int SMEM = 1024 + OFF_BAR + 256;
  static constexpr uint32_t TMEM_COLS = 256;  // S: [0,128), O: [128, 128+DH)
};

__device__ __forceinline__ void fa_keep128(uint64_t seed, uint32_t layer, uint64_t row, int key0, uint32_t thresh,
                                           uint32_t (&bits)[4]) {
  // 128 keep bits (keys key0 .. key0+127) of one probability row, 16 Philox calls
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t word = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      bool k8[8];
      dropout_keep8(seed, layer, 0u, row, key0 + w * 32 + c * 8, thresh, k8);
#pragma unroll
      for (int e = 0; e < 8; ++e) word |= (k8[e] ? 1u : 0u) << (c * 8 + e);
    }
    bits[w] = word;
  }
}

template <int DH>
__global__ void __launch_bounds__(FA_THREADS, (DH == 64 ? 2 : 1))
    flash_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const FaFwdArgs a) {
  using Cfg = FaFwdCfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;   // [2]
  uint64_t* kv_empty = bar + 3;  // [2]
  uint64_t* s_full = bar + 5;
  uint64_t* s_free = bar + 6;
  uint64_t* p_full = bar + 7;
  uint64_t* o_done = bar + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = (a.s + FA_BQ - 1) / FA_BQ;
  const int qt = n_qt - 1 - (int)blockIdx.x;  // heavy (causal) tiles first
  const int h = blockIdx.y, b = blockIdx.z;
  const int n_kt = a.causal ? (qt + 1) : (a.s + FA_BK - 1) / FA_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 128);
    mbar_init(p_full, 128);
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_arrive_expect_tx(q_full, Cfg::Q_BYTES);
#pragma unroll
      for (int kb = 0; kb < DH / 64; ++kb)
        tma_load_4d(smem + Cfg::OFF_Q + kb * (FA_BQ * 128), &tmQ, q_full, kb * 64, qt * FA_BQ, h, b);
      for (int j = 0; j < n_kt; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], Cfg::K_BYTES + Cfg::V_BYTES);
        uint8_t* k_dst = smem + Cfg::OFF_K + st * Cfg::K_BYTES;
        uint8_t* v_dst = smem + Cfg::OFF_V + st * Cfg::V_BYTES;
#pragma unroll
        for (int kb = 0; kb < DH / 64; ++kb)
          tma_load_4d(k_dst + kb * (FA_BK * 128), &tmK, &kv_full[st], kb * 64, j * FA_BK, h, b);
        // V as the MN-major B operand of P.V: [64-key block][64-wide d chunk][64 keys x 128 B]
#pragma unroll
        for (int kb = 0; kb < FA_BK / 64; ++kb)
#pragma unroll
          for (int c = 0; c < DH / 64; ++c)
            tma_load_4d(v_dst + (kb * (DH / 64) + c) * 8192, &tmV, &kv_full[st], c * 64, j * FA_BK + kb * 64, h, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t idS = make_idesc_bf16(128, FA_BK, false, false);
      const uint32_t idO = make_idesc_bf16(128, DH, false, true);
      const uint32_t q_base = smem_u32(smem + Cfg::OFF_Q);
      const uint32_t p_base = smem_u32(smem + Cfg::OFF_P);
      mbar_wait(q_full, 0);
      for (int j = 0; j <= n_kt; ++j) {
        if (j < n_kt) {
          const int st = j & 1;
          mbar_wait(&kv_full[st], (j >> 1) & 1);
          if (j > 0) mbar_wait(s_free, (j - 1) & 1);  // softmax has read S_{j-1}
          tc_fence_after();
          const uint32_t k_base = smem_u32(smem + Cfg::OFF_K + st * Cfg::K_BYTES);
#pragma unroll
          for (int kb = 0; kb < DH / 64; ++kb)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tS, make_sw128_desc(q_base + kb * (FA_BQ * 128) + k * 32, 16, 1024),
                        make_sw128_desc(k_base + kb * (FA_BK * 128) + k * 32, 16, 1024), idS, (kb | k) != 0);
          umma_commit(s_full);
        }
        if (j > 0) {
          const int jp = j - 1, st = jp & 1;
          mbar_wait(p_full, jp & 1);  // P_{j-1} in smem, O rescaled
          tc_fence_after();
          const uint32_t v_base = smem_u32(smem + Cfg::OFF_V + st * Cfg::V_BYTES);
#pragma unroll
          for (int kb = 0; kb < FA_BK / 64; ++kb)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tO, make_sw128_desc(p_base + kb * (FA_BQ * 128) + k * 32, 16, 1024),
                        make_sw128_desc(v_base + kb * (DH / 64) * 8192 + k * 2048, 8192, 1024), idO,
                        (jp > 0) || ((kb | k) != 0));
          umma_commit(o_done);
          umma_commit(&kv_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax / epilogue (thread = query row) ----------------
    const int r = (warp - 4) * 32 + lane;  // row within tile == TMEM lane
    const int q = qt * FA_BQ + r;
    const uint32_t t_lane = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const float* mrow = a.mask ? a.mask + (int64_t)b * a.s : nullptr;
    const uint64_t prow = (uint64_t)(((a.sample_offset + b) * a.nh_global + a.head_offset + h) * (int64_t)a.s + q);
    uint8_t* p_smem = smem + Cfg::OFF_P;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kt; ++j) {
      const int key0 = j * FA_BK;
      const bool diag = a.causal && (j == qt);
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      // pass 1: row max of the scaled, masked scores (read TMEM 32 columns at a time)
      float mx = -INFINITY;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tS + t_lane + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int key = key0 + c * 32 + e;
          float x = __uint_as_float(v[e]) * a.scale_log2;
          if (mrow) x += __ldg(mrow + key) * 1.4426950408889634f;
          if ((diag && key > q) || key >= a.s) x = -INFINITY;
          mx = fmaxf(mx, x);
        }
      }
      const float m_new = fmaxf(m, mx);
      const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
      const float alpha = (m == -INFINITY) ? 0.f : ex2_approx(m - m_use);
      uint32_t keep[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
      if (a.p > 0.f) fa_keep128(a.seed, a.layer, prow, key0, a.thresh, keep);
      if (j > 0) {
        // P.V of tile j-1 must have finished: it reads the P buffer we overwrite below
        // and accumulates into the O we rescale
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
        if (!__all_sync(0xffffffffu, alpha == 1.f)) {
#pragma unroll
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + t_lane + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st_32x32b_x32(tO + t_lane + c * 32, o);
          }
          tmem_st_wait();
        }
      }
      // pass 2: p = exp2(x - m); row sum; dropout; bf16 P -> smem as the swizzled K-major
      // A operand (keys [64kb, 64kb+64) in sub-tile kb; 16-B granule g = keys 8g..8g+7)
      float rowsum = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tS + t_lane + c * 32, v);
        tmem_ld_wait();
        if (c == 3) {
          tc_fence_before();
          mbar_arrive(s_free);  // S fully read: the MMA warp may overwrite it
        }
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float pe[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int key = key0 + c * 32 + e + u;
            float x = __uint_as_float(v[e + u]) * a.scale_log2;
            if (mrow) x += __ldg(mrow + key) * 1.4426950408889634f;
            if ((diag && key > q) || key >= a.s) x = -INFINITY;
            const float pr = ex2_approx(x - m_use);
            rowsum += pr;
            pe[u] = ((keep[c] >> (e + u)) & 1u) ? pr * a.inv_keep : 0.f;
          }
          pk[e / 2] = pack_bf16x2(pe[0], pe[1]);
        }
        const int kb = c >> 1;
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) {
          const int g = (c & 1) * 4 + gg;
          *reinterpret_cast<uint4*>(p_smem + kb * (FA_BQ * 128) + sw128_offset(r, g)) =
              make_uint4(pk[gg * 4], pk[gg * 4 + 1], pk[gg * 4 + 2], pk[gg * 4 + 3]);
        }
      }
      l = l * alpha + rowsum;
      m = m_new;
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16; lse
    mbar_wait(o_done, (n_kt - 1) & 1);
    tc_fence_after();
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    bf16* orow = a.out + ((int64_t)b * a.s + q) * a.ld_out + (int64_t)h * DH;
#pragma unroll
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tO + t_lane + c * 32, o);
      tmem_ld_wait();
      if (q < a.s) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint4 u;
          u.x = pack_bf16x2(__uint_as_float(o[g * 8 + 0]) * inv_l, __uint_as_float(o[g * 8 + 1]) * inv_l);
          u.y = pack_bf16x2(__uint_as_float(o[g * 8 + 2]) * inv_l, __uint_as_float(o[g * 8 + 3]) * inv_l);
          u.z = pack_bf16x2(__uint_as_float(o[g * 8 + 4]) * inv_l, __uint_as_float(o[g * 8 + 5]) * inv_l);
          u.w = pack_bf16x2(__uint_as_float(o[g * 8 + 6]) * inv_l, __uint_as_float(o[g * 8 + 7]) * inv_l);
          *reinterpret_cast<uint4*>(orow + c * 32 + g * 8) = u;
        }
      }
    }
    if (q < a.s && a.lse) a.lse[((int64_t)b * a.nh + h) * a.s + q] = (l > 0.f) ? m + __log2f(l) : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, Cfg::TMEM_COLS);
  }
}

}  // namespace smpk

using namespace smpk;

// defined in gemm.cu
namespace smpk {
int make_tma_4d(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int nb1, int64_t s1,
                int nb2, int64_t s2, int box_inner, int box_outer, const char* name);
}

extern "C" int smpk_flash_attn_fwd(const void* qkv, int64_t ld, int B, int nh, int s, int dh, void* out,
                                   int64_t ld_out, float* lse, const float* mask_add, float scale, int causal,
                                   float p_drop, uint64_t seed, int layer, int64_t sample_offset, int head_offset,
                                   int nh_global, void* stream) {
  SMPK_REQUIRE(dh == 64 || dh == 128, SMPK_ERR_UNSUPPORTED, "smpk_flash_attn_fwd: head dim %d (64 or 128)", dh);
  SMPK_REQUIRE(s % 128 == 0 && s > 0, SMPK_ERR_UNSUPPORTED, "smpk_flash_attn_fwd: seq %d must be a multiple of 128",
               s);
  SMPK_REQUIRE(qkv && out && B > 0 && nh > 0, SMPK_ERR_BAD_ARG, "smpk_flash_attn_fwd: bad arguments");
  SMPK_REQUIRE(p_drop >= 0.f && p_drop < 1.f, SMPK_ERR_BAD_ARG, "smpk_flash_attn_fwd: dropout p in [0,1)");
  SMPK_REQUIRE(ld_out % 8 == 0, SMPK_ERR_BAD_ARG, "smpk_flash_attn_fwd: ld_out must be a multiple of 8");
  const int64_t hd = (int64_t)nh * dh;
  const bf16* base = reinterpret_cast<const bf16*>(qkv);
  CUtensorMap tq, tk, tv;
  int rc = make_tma_4d(&tq, base, dh, s, ld, nh, dh, B, (int64_t)s * ld, 64, 128, "Q");
  if (!rc) rc = make_tma_4d(&tk, base + hd, dh, s, ld, nh, dh, B, (int64_t)s * ld, 64, 128, "K");
  if (!rc) rc = make_tma_4d(&tv, base + 2 * hd, dh, s, ld, nh, dh, B, (int64_t)s * ld, 64, 64, "V");
  if (rc) return rc;
  FaFwdArgs a;
  a.B = B;
  a.nh = nh;
  a.s = s;
  a.out = reinterpret_cast<bf16*>(out);
  a.ld_out = ld_out;
  a.lse = lse;
  a.mask = mask_add;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.causal = causal;
  a.p = p_drop;
  a.inv_keep = p_drop > 0.f ? 1.f / (1.f - p_drop) : 1.f;
  a.thresh = dropout_threshold(p_drop);
  a.seed = seed;
  a.layer = (uint32_t)layer;
  a.sample_offset = sample_offset;
  a.head_offset = head_offset;
  a.nh_global = nh_global;
  dim3 grid(s / 128, nh, B);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dh == 64) {
    static bool once = false;
    if (!once) {
      cudaFuncSetAttribute(flash_fwd_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, FaFwdCfg<64>::SMEM);
      once = true;
    }
    flash_fwd_kernel<64><<<grid, FA_THREADS, FaFwdCfg<64>::SMEM, st>>>(tq, tk, tv, a);
  } else {
    static bool once = false;
    if (!once) {
      cudaFuncSetAttribute(flash_fwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, FaFwdCfg<128>::SMEM);
      once = true;
    }
    flash_fwd_kernel<128><<<grid, FA_THREADS, FaFwdCfg<128>::SMEM, st>>>(tq, tk, tv, a);
  }
  return check_launch("smpk_flash_attn_fwd");
}

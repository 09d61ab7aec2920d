// flash_attn_bwd.cu — fused attention backward on tcgen05/TMEM/TMA (sm_100a).
//
// CTA = (128-key tile j, local head, sample); it keeps K_j, V_j in smem and the dK, dV
// accumulators in TMEM while streaming the query tiles i (i >= j when causal):
//   (a) S^T  = K_j Q_i^T           (M=keys, N=queries, K=dh)      -> TMEM
//   (b) dP^T = V_j dO_i^T          (M=keys, N=queries, K=dh)      -> TMEM
//   softmax-backward warps (thread = key row):
//       P  = exp2(S*scale*log2e + mask - lse2[q])   (recomputed, never stored in HBM)
//       Pd = P * keep / (1-p)  -> smem (K-major A operand)
//       dS = P * (dP - Delta[q]),  dP = dPd * keep / (1-p)  -> smem
//   (c) dV += Pd^T dO_i            (A = Pd^T K-major, B = dO_i read MN-major)
//   (d) dK += dS^T Q_i             (A = dS^T K-major, B = Q_i  read MN-major)
//   (e) dQ_i(j) = dS K_j           (A = dS^T read MN-major, B = K_j read MN-major) -> TMEM
//       drained as an fp32 partial per key tile; smpk_flash_dq_reduce sums the partials
//       in key-tile order (bit-deterministic, no float atomics).
// The same K-major SWIZZLE_128B smem tile of Q / dO / K / dS serves both as a K-major and
// (through a different UMMA descriptor) as an MN-major operand.
// Dropout keep bits are generated row-wise (thread = query row, 16 Philox calls per tile,
// exactly the forward's stream) into a shared bitmask and read column-wise.
#include "smpk_common.cuh"

namespace smpk {

int make_tma_4d(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int nb1, int64_t s1,
                int nb2, int64_t s2, int box_inner, int box_outer, const char* name);

constexpr int FB_THREADS = 256;

struct FaBwdArgs {
  int B, nh, s;
  const float* lse;    // [B, nh, s] log2 domain (from the forward)
  const float* delta;  // [B, nh, s] rowsum(dO * O)
  const float* mask;   // [B, s] additive or null
  float scale_log2, scale;
  int causal;
  float p, inv_keep;
  uint32_t thresh;
  uint64_t seed;
  uint32_t layer;
  int64_t sample_offset;
  int head_offset, nh_global;
  bf16* dqkv;
  int64_t ld;  // of qkv / dqkv
  int64_t H;   // nh * dh
  float* dq_part;  // [n_kt][B*s][H]
};

template <int DH>
struct FaBwdCfg {
  static constexpr int NST = DH == 64 ? 2 : 1;
  static constexpr int TILE = 128 * DH * 2;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + TILE;
  static constexpr int OFF_Q = OFF_V + TILE;
  static constexpr int OFF_DO = OFF_Q + NST * TILE;
  static constexpr int OFF_PDT = OFF_DO + NST * TILE;
  static constexpr int OFF_DST = OFF_PDT + 32768;
  static constexpr int OFF_LSE = OFF_DST + 32768;
  static constexpr int OFF_DELTA = OFF_LSE + NST * 512;
  static constexpr int OFF_BITS = OFF_DELTA + NST * 512;
  static constexpr int OFF_BAR = OFF_BITS + 2 * 128 * 4 * 4;
  static constexpr int SMEM = 1024 + OFF_BAR + 256;
  // TMEM: S^T / dQ [0,128), dP^T [128,256), dV [256, 256+DH), dK [256+DH, 256+2DH)
  static constexpr uint32_t TMEM_COLS = 512;
};

__device__ __forceinline__ void fb_keep128(uint64_t seed, uint32_t layer, uint64_t row, int key0, uint32_t thresh,
                                           uint32_t* out4) {
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
    out4[w] = word;
  }
}

template <int DH>
__global__ void __launch_bounds__(FB_THREADS, 1)
    flash_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                     const FaBwdArgs a) {
  using Cfg = FaBwdCfg<DH>;
  constexpr int NST = Cfg::NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* qdo_full = bar + 1;   // [2]
  uint64_t* qdo_empty = bar + 3;  // [2]
  uint64_t* st_full = bar + 5;
  uint64_t* pdt_full = bar + 6;
  uint64_t* dst_full = bar + 7;
  uint64_t* mma_done = bar + 8;
  uint64_t* dq_free = bar + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 11);

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
    mbar_init(kv_full, 1);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&qdo_full[x], 1);
      mbar_init(&qdo_empty[x], 1);
    }
    mbar_init(st_full, 1);
    mbar_init(pdt_full, 128);
    mbar_init(dst_full, 128);
    mbar_init(mma_done, 1);
    mbar_init(dq_free, 128);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 256 + DH;

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
        const int i = i0 + t, stg = t % NST;
        mbar_wait(&qdo_empty[stg], ((t / NST) & 1) ^ 1);
        mbar_arrive_expect_tx(&qdo_full[stg], 2 * Cfg::TILE + 1024);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c) {
          tma_load_4d(smem + Cfg::OFF_Q + stg * Cfg::TILE + c * 16384, &tmQ, &qdo_full[stg], c * 64, i * 128, h, b);
          tma_load_4d(smem + Cfg::OFF_DO + stg * Cfg::TILE + c * 16384, &tmDO, &qdo_full[stg], c * 64, i * 128, h,
                      b);
        }
        const int64_t off = ((int64_t)b * a.nh + h) * a.s + (int64_t)i * 128;
        bulk_load(smem + Cfg::OFF_LSE + stg * 512, a.lse + off, 512, &qdo_full[stg]);
        bulk_load(smem + Cfg::OFF_DELTA + stg * 512, a.delta + off, 512, &qdo_full[stg]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t idKK = make_idesc_bf16(128, 128, false, false);
      const uint32_t idKM = make_idesc_bf16(128, DH, false, true);
      const uint32_t idMM = make_idesc_bf16(128, DH, true, true);
      const uint32_t k_base = smem_u32(smem + Cfg::OFF_K), v_base = smem_u32(smem + Cfg::OFF_V);
      const uint32_t pdt = smem_u32(smem + Cfg::OFF_PDT), dst = smem_u32(smem + Cfg::OFF_DST);
      mbar_wait(kv_full, 0);
      for (int t = 0; t < nt; ++t) {
        const int stg = t % NST;
        const uint32_t q_base = smem_u32(smem + Cfg::OFF_Q + stg * Cfg::TILE);
        const uint32_t do_base = smem_u32(smem + Cfg::OFF_DO + stg * Cfg::TILE);
        mbar_wait(&qdo_full[stg], (t / NST) & 1);
        if (t > 0) mbar_wait(dq_free, (t - 1) & 1);  // dQ_{t-1} drained: S^T region free
        tc_fence_after();
        // (a) S^T = K Q^T, (b) dP^T = V dO^T
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            umma_bf16(tS, make_sw128_desc(k_base + c * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(q_base + c * 16384 + k * 32, 16, 1024), idKK, (c | k) != 0);
            umma_bf16(tdP, make_sw128_desc(v_base + c * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(do_base + c * 16384 + k * 32, 16, 1024), idKK, (c | k) != 0);
          }
        umma_commit(st_full);
        // (c) dV += Pd^T dO
        mbar_wait(pdt_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tdV, make_sw128_desc(pdt + kb * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(do_base + kb * 8192 + k * 2048, 16384, 1024), idKM, (t > 0) || ((kb | k) != 0));
        // (d) dK += dS^T Q ; (e) dQ = dS K
        mbar_wait(dst_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            umma_bf16(tdK, make_sw128_desc(dst + kb * 16384 + k * 32, 16, 1024),
                      make_sw128_desc(q_base + kb * 8192 + k * 2048, 16384, 1024), idKM, (t > 0) || ((kb | k) != 0));
            umma_bf16(tS, make_sw128_desc(dst + kb * 8192 + k * 2048, 16384, 1024),
                      make_sw128_desc(k_base + kb * 8192 + k * 2048, 16384, 1024), idMM, (kb | k) != 0);
          }
        umma_commit(mma_done);
        umma_commit(&qdo_empty[stg]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax backward (thread = key row r) ----------------
    const int r = (warp - 4) * 32 + lane;
    const int key = j * 128 + r;
    const uint32_t t_lane = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const float mk = a.mask ? a.mask[(int64_t)b * a.s + key] * 1.4426950408889634f : 0.f;
    uint8_t* pdt_s = smem + Cfg::OFF_PDT;
    uint8_t* dst_s = smem + Cfg::OFF_DST;
    uint32_t* bits = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BITS);
    const int64_t prow0 = ((a.sample_offset + b) * a.nh_global + a.head_offset + h) * (int64_t)a.s;
    for (int t = 0; t < nt; ++t) {
      const int i = i0 + t, stg = t % NST;
      const bool diag = a.causal && (i == j);
      const float* lse_s = reinterpret_cast<const float*>(smem + Cfg::OFF_LSE + stg * 512);
      const float* del_s = reinterpret_cast<const float*>(smem + Cfg::OFF_DELTA + stg * 512);
      uint32_t* bt = bits + (t & 1) * 512;
      if (a.p > 0.f) {
        // this thread generates the keep bits of query row i*128 + r (forward's Philox stream)
        fb_keep128(a.seed, a.layer, (uint64_t)(prow0 + (int64_t)i * 128 + r), j * 128, a.thresh, bt + r * 4);
        named_barrier_sync(1, 128);
      }
      mbar_wait(&qdo_full[stg], (t / NST) & 1);  // lse / delta of this query tile in smem
      mbar_wait(st_full, t & 1);
      tc_fence_after();
      // pass A: Pd^T row -> smem
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t sv[32];
        tmem_ld_32x32b_x32(tS + t_lane + c * 32, sv);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float pd[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int qq = c * 32 + e + u;
            const float l2 = lse_s[qq];
            float x = __uint_as_float(sv[e + u]) * a.scale_log2 + mk - l2;
            float pr = (l2 == -INFINITY || (diag && r > qq)) ? 0.f : ex2_approx(x);
            bool kp = true;
            if (a.p > 0.f) kp = (bt[qq * 4 + (r >> 5)] >> (r & 31)) & 1u;
            pd[u] = kp ? pr * a.inv_keep : 0.f;
          }
          pk[e / 2] = pack_bf16x2(pd[0], pd[1]);
        }
        const int kb = c >> 1;
#pragma unroll
        for (int gg = 0; gg < 4; ++gg)
          *reinterpret_cast<uint4*>(pdt_s + kb * 16384 + sw128_offset(r, (c & 1) * 4 + gg)) =
              make_uint4(pk[gg * 4], pk[gg * 4 + 1], pk[gg * 4 + 2], pk[gg * 4 + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(pdt_full);
      // pass B: dS^T row -> smem
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t sv[32], dv[32];
        tmem_ld_32x32b_x32(tS + t_lane + c * 32, sv);
        tmem_ld_32x32b_x32(tdP + t_lane + c * 32, dv);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float ds[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int qq = c * 32 + e + u;
            const float l2 = lse_s[qq];
            float x = __uint_as_float(sv[e + u]) * a.scale_log2 + mk - l2;
            float pr = (l2 == -INFINITY || (diag && r > qq)) ? 0.f : ex2_approx(x);
            bool kp = true;
            if (a.p > 0.f) kp = (bt[qq * 4 + (r >> 5)] >> (r & 31)) & 1u;
            const float dp = kp ? __uint_as_float(dv[e + u]) * a.inv_keep : 0.f;
            ds[u] = pr * (dp - del_s[qq]);
          }
          pk[e / 2] = pack_bf16x2(ds[0], ds[1]);
        }
        const int kb = c >> 1;
#pragma unroll
        for (int gg = 0; gg < 4; ++gg)
          *reinterpret_cast<uint4*>(dst_s + kb * 16384 + sw128_offset(r, (c & 1) * 4 + gg)) =
              make_uint4(pk[gg * 4], pk[gg * 4 + 1], pk[gg * 4 + 2], pk[gg * 4 + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(dst_full);
      // drain dQ_i(j) (thread = query row r) as an fp32 partial
      mbar_wait(mma_done, t & 1);
      tc_fence_after();
      float* dq = a.dq_part + ((int64_t)j * a.B * a.s + (int64_t)b * a.s + (int64_t)i * 128 + r) * a.H +
                  (int64_t)h * DH;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tS + t_lane + c * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 8; ++g)
          *reinterpret_cast<float4*>(dq + c * 32 + g * 4) =
              make_float4(__uint_as_float(o[g * 4]) * a.scale, __uint_as_float(o[g * 4 + 1]) * a.scale,
                          __uint_as_float(o[g * 4 + 2]) * a.scale, __uint_as_float(o[g * 4 + 3]) * a.scale);
      }
      tc_fence_before();
      mbar_arrive(dq_free);
    }
    // dK (scaled) and dV rows of this key tile -> dqkv (bf16)
    bf16* dkrow = a.dqkv + ((int64_t)b * a.s + key) * a.ld + a.H + (int64_t)h * DH;
    bf16* dvrow = dkrow + a.H;
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
        uv.x = pack_bf16x2(__uint_as_float(vv[g * 8 + 0]), __uint_as_float(vv[g * 8 + 1]));
        uv.y = pack_bf16x2(__uint_as_float(vv[g * 8 + 2]), __uint_as_float(vv[g * 8 + 3]));
        uv.z = pack_bf16x2(__uint_as_float(vv[g * 8 + 4]), __uint_as_float(vv[g * 8 + 5]));
        uv.w = pack_bf16x2(__uint_as_float(vv[g * 8 + 6]), __uint_as_float(vv[g * 8 + 7]));
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

// Delta[b, h, q] = sum_d dO[b*s+q, h*dh+d] * O[b*s+q, h*dh+d]   (one thread per (row, head))
__global__ void flash_delta_kernel(const bf16* __restrict__ o, int64_t ld_o, const bf16* __restrict__ dout,
                                   int64_t ld_do, int B, int nh, int s, int dh, float* __restrict__ delta) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)B * s * nh;
  if (idx >= total) return;
  const int h = (int)(idx % nh);
  const int64_t row = idx / nh;
  const bf16* op = o + row * ld_o + (int64_t)h * dh;
  const bf16* dp = dout + row * ld_do + (int64_t)h * dh;
  float acc = 0.f;
  for (int d = 0; d < dh; d += 8) {
    uint4 a = *reinterpret_cast<const uint4*>(op + d);
    uint4 c = *reinterpret_cast<const uint4*>(dp + d);
    uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 fa = unpack_bf16x2(wa[k]), fc = unpack_bf16x2(wc[k]);
      acc += fa.x * fc.x + fa.y * fc.y;
    }
  }
  const int64_t b = row / s, q = row % s;
  delta[(b * nh + h) * s + q] = acc;
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

extern "C" int64_t smpk_flash_attn_bwd_workspace(int B, int nh, int s, int dh) {
  const int64_t n_kt = s / 128;
  return n_kt * (int64_t)B * s * nh * dh * 4 + (int64_t)B * nh * s * 4;
}

extern "C" int smpk_flash_attn_bwd(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* dout,
                                   int64_t ld_dout, const float* lse, int B, int nh, int s, int dh, void* dqkv,
                                   const float* mask_add, float scale, int causal, float p_drop, uint64_t seed,
                                   int layer, int64_t sample_offset, int head_offset, int nh_global, void* workspace,
                                   int64_t workspace_bytes, void* stream) {
  SMPK_REQUIRE(dh == 64 || dh == 128, SMPK_ERR_UNSUPPORTED, "smpk_flash_attn_bwd: head dim %d (64 or 128)", dh);
  SMPK_REQUIRE(s % 128 == 0 && s > 0, SMPK_ERR_UNSUPPORTED, "smpk_flash_attn_bwd: seq %d must be a multiple of 128",
               s);
  SMPK_REQUIRE(qkv && out && dout && lse && dqkv, SMPK_ERR_BAD_ARG, "smpk_flash_attn_bwd: null argument");
  SMPK_REQUIRE(ld % 8 == 0 && ld_out % 8 == 0 && ld_dout % 8 == 0, SMPK_ERR_BAD_ARG,
               "smpk_flash_attn_bwd: leading dims must be multiples of 8");
  const int64_t need = smpk_flash_attn_bwd_workspace(B, nh, s, dh);
  SMPK_REQUIRE(workspace && workspace_bytes >= need, SMPK_ERR_BAD_ARG, "smpk_flash_attn_bwd: workspace too small");
  const int64_t H = (int64_t)nh * dh;
  const int n_kt = s / 128;
  float* dq_part = reinterpret_cast<float*>(workspace);
  float* delta = dq_part + (int64_t)n_kt * B * s * H;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  {
    const int64_t total = (int64_t)B * s * nh;
    flash_delta_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const bf16*>(out), ld_out, reinterpret_cast<const bf16*>(dout), ld_dout, B, nh, s, dh,
        delta);
    int rc = check_launch("smpk_flash_attn_bwd(delta)");
    if (rc) return rc;
  }
  const bf16* base = reinterpret_cast<const bf16*>(qkv);
  CUtensorMap tq, tk, tv, tdo;
  int rc = make_tma_4d(&tq, base, dh, s, ld, nh, dh, B, (int64_t)s * ld, 64, 128, "Q");
  if (!rc) rc = make_tma_4d(&tk, base + H, dh, s, ld, nh, dh, B, (int64_t)s * ld, 64, 128, "K");
  if (!rc) rc = make_tma_4d(&tv, base + 2 * H, dh, s, ld, nh, dh, B, (int64_t)s * ld, 64, 128, "V");
  if (!rc) rc = make_tma_4d(&tdo, dout, dh, s, ld_dout, nh, dh, B, (int64_t)s * ld_dout, 64, 128, "dO");
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
  a.p = p_drop;
  a.inv_keep = p_drop > 0.f ? 1.f / (1.f - p_drop) : 1.f;
  a.thresh = dropout_threshold(p_drop);
  a.seed = seed;
  a.layer = (uint32_t)layer;
  a.sample_offset = sample_offset;
  a.head_offset = head_offset;
  a.nh_global = nh_global;
  a.dqkv = reinterpret_cast<bf16*>(dqkv);
  a.ld = ld;
  a.H = H;
  a.dq_part = dq_part;
  dim3 grid(n_kt, nh, B);
  if (dh == 64) {
    static bool once = false;
    if (!once) {
      cudaFuncSetAttribute(flash_bwd_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, FaBwdCfg<64>::SMEM);
      once = true;
    }
    flash_bwd_kernel<64><<<grid, FB_THREADS, FaBwdCfg<64>::SMEM, st>>>(tq, tk, tv, tdo, a);
  } else {
    static bool once = false;
    if (!once) {
      cudaFuncSetAttribute(flash_bwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, FaBwdCfg<128>::SMEM);
      once = true;
    }
    flash_bwd_kernel<128><<<grid, FB_THREADS, FaBwdCfg<128>::SMEM, st>>>(tq, tk, tv, tdo, a);
  }
  rc = check_launch("smpk_flash_attn_bwd");
  if (rc) return rc;
  const int64_t n4 = (int64_t)B * s * H / 4;
  flash_dq_reduce_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(dq_part, n_kt, (int64_t)B * s, H, s, causal,
                                                                      reinterpret_cast<bf16*>(dqkv), ld);
  return check_launch("smpk_flash_attn_bwd(dq reduce)");
}

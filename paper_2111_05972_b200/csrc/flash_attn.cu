// flash_attn.cu — fused attention forward on tcgen05/TMEM/TMA (sm_100a), and the
// attention-dropout keep-bit generator shared by the forward and the backward.
//
// The attention core of dist_attention_forward for one TP rank's
// local heads: softmax(Q K^T / sqrt(dh) + mask [+ causal]) -> dropout -> . V, without
// materialising the [s, s] score / probability matrices in HBM.
//
// CTA = two 128-row query tiles (Q0, Q1) of one (head, sample); 384 threads:
//   warp 0      TMA producer: Q0/Q1 once, K/V tiles through an NS-stage ring (shared by
//               both query tiles, so K/V are read once per 256 queries)
//   warp 1      MMA issuer (whole warp, one elected lane issues):
//                 S_t = Q_t K_j^T (M=128, N=128) into TMEM;  O_t += P_t V_j (M=128, N=dh)
//               ping-pong order  PV0_j, S0_{j+1}, PV1_j, S1_{j+1}  so each softmax group
//               gets its next scores while the other one computes
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O0 | O1)
//   warps 4-7   softmax group 0 (query tile Q0), warps 8-11 softmax group 1 (Q1):
//               thread = query row = TMEM lane; the 128 scores of the row are read once
//               into registers; online max / sum in the exp2 domain; O rescaled in TMEM
//               only when some row's running max grew; dropout from precomputed keep bits
//               (smpk_attn_dropout_bits, the Philox stream of oracle/philox.py); P written to
//               smem as the swizzled K-major A operand of P.V; 1/(1-p) and 1/l applied once
//               in the epilogue.
#include "smpk_common.cuh"

namespace smpk {

int make_tma_4d(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int nb1, int64_t s1,
                int nb2, int64_t s2, int box_inner, int box_outer, const char* name);

constexpr int FA_THREADS = 384;
constexpr int FA_BQ = 128;
constexpr int FA_BK = 128;

struct FaFwdArgs {
  int B, nh, s;
  bf16* out;
  int64_t ld_out;
  float* lse;                // [B, nh, s] log2-domain log-sum-exp of the scaled+masked scores
  const float* mask;         // [B, s] additive, may be null
  const uint32_t* keep;      // [B, nh, s, s/32] dropout keep bits (null: no dropout)
  float scale_log2;          // log2(e) / sqrt(dh)
  int causal;
  float inv_keep;
  int trace;
};

// K and V stream through separate rings: K_{j+1} only has to wait for both tiles' S_j, V_{j+1}
// for both tiles' P_j.V_j -- at dh = 128 (no room for two full K/V stages next to P) K is double
// buffered and V single buffered, so the next K load overlaps the current tile's softmax.
template <int DH, int NS_ = (DH == 64 ? 3 : 2), int NSV_ = (DH == 64 ? 3 : 1)>
struct FaFwdCfg {
  static constexpr int NS = NS_;    // K ring depth
  static constexpr int NSV = NSV_;  // V ring depth
  static constexpr int Q_BYTES = FA_BQ * DH * 2;
  static constexpr int K_BYTES = FA_BK * DH * 2;
  static constexpr int V_BYTES = FA_BK * DH * 2;
  static constexpr int P_BYTES = FA_BQ * FA_BK * 2;
  static constexpr int OFF_Q = 0;                          // Q0, Q1
  static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + NS * K_BYTES;
  static constexpr int OFF_P = OFF_V + NSV * V_BYTES;      // P0, P1
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int SMEM = 1024 + OFF_BAR + 256;
  static constexpr uint32_t TMEM_COLS = 512;  // S0 [0,128) S1 [128,256) O0 [256,256+DH) O1 [256+DH, 256+2DH)
};

// debug timeline (SMPK_FA_TRACE=1): per CTA [0] start [1] Q landed (MMA warp) [2..9] group-0 S_j ready
// [10..17] group-0 P_j stored [18] epilogue done (group 0) [19] %smid
__device__ unsigned long long g_fa_trace[1024 * 20];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int DH, int NS_, int NSV_>
__global__ void __launch_bounds__(FA_THREADS, 1)
    flash_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const FaFwdArgs a) {
  using Cfg = FaFwdCfg<DH, NS_, NSV_>;
  constexpr int NSV = Cfg::NSV;
  constexpr int NS = Cfg::NS;
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ array (not an integer round trip) keeps the shared
  // address space visible to the compiler: LDS / STS instead of generic LD / ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  static_assert(NS <= 4 && NSV <= 4, "K/V ring depth");
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;        // [NS]  K ring
  uint64_t* kv_empty = bar + 5;       // [NS]
  uint64_t* v_full = bar + 9;         // [NSV] V ring
  uint64_t* v_empty = bar + 13;       // [NSV]
  uint64_t* s_full = bar + 17;        // [2]
  uint64_t* p_full = bar + 19;        // [2]
  uint64_t* o_done = bar + 21;        // [2]
  uint64_t* s_read = bar + 23;        // [2] softmax group t has loaded S_t into registers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 25);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = a.s / FA_BQ;
  const int n_kv = a.s / FA_BK;
  const int qt0 = 2 * (int)blockIdx.x;
  const int nq = min(2, n_qt - qt0);  // query tiles of this CTA
  const int h = blockIdx.y, b = blockIdx.z;
  // key tiles each query tile needs, and the iteration count of the shared K/V stream
  const int nkt0 = a.causal ? qt0 + 1 : n_kv;
  const int nkt1 = nq > 1 ? (a.causal ? qt0 + 2 : n_kv) : 0;
  const int n_iter = max(nkt0, nkt1);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < NSV; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 4);  // one arrive per softmax warp
      mbar_init(&o_done[t], 1);
      mbar_init(&s_read[t], 4);  // one arrive per softmax warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  const int cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  unsigned long long* trc = (a.trace && cta_lin < 1024) ? g_fa_trace + cta_lin * 20 : nullptr;
  if (trc && threadIdx.x == 0) {
    trc[0] = gtime();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    trc[19] = smid;
  }

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: Q, then the K ring ----------------
      mbar_arrive_expect_tx(q_full, nq * Cfg::Q_BYTES);
      for (int t = 0; t < nq; ++t)
#pragma unroll
        for (int kb = 0; kb < DH / 64; ++kb)
          tma_load_4d(smem + Cfg::OFF_Q + t * Cfg::Q_BYTES + kb * (FA_BQ * 128), &tmQ, q_full, kb * 64,
                      (qt0 + t) * FA_BQ, h, b);
      for (int j = 0; j < n_iter; ++j) {
        const int st = j % NS;
        mbar_wait(&kv_empty[st], ((j / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], Cfg::K_BYTES);
        uint8_t* k_dst = smem + Cfg::OFF_K + st * Cfg::K_BYTES;
#pragma unroll
        for (int kb = 0; kb < DH / 64; ++kb)
          tma_load_4d(k_dst + kb * (FA_BK * 128), &tmK, &kv_full[st], kb * 64, j * FA_BK, h, b);
      }
    } else if (lane == 1) {
      // ---------------- TMA producer: the V ring ----------------
      for (int j = 0; j < n_iter; ++j) {
        const int st = j % NSV;
        mbar_wait(&v_empty[st], ((j / NSV) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[st], Cfg::V_BYTES);
        uint8_t* v_dst = smem + Cfg::OFF_V + st * Cfg::V_BYTES;
        // V as the MN-major B operand of P.V: [64-key block][64-wide d chunk][64 keys x 128 B]
#pragma unroll
        for (int kb = 0; kb < FA_BK / 64; ++kb)
#pragma unroll
          for (int c = 0; c < DH / 64; ++c)
            tma_load_4d(v_dst + (kb * (DH / 64) + c) * 8192, &tmV, &v_full[st], c * 64, j * FA_BK + kb * 64, h, b);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp; one elected lane issues) ----------------
    // Event-driven: S_t(j+1) is issued as soon as softmax group t has READ S_t(j) into registers
    // (s_read), so the next scores are computed while the group is still exponentiating; P_t(j).V_j
    // follows p_full.  Both groups' events are polled, so neither waits behind the other's phase.
    const uint32_t idS = make_idesc_bf16(128, FA_BK, false, false);
    const uint32_t idO = make_idesc_bf16(128, DH, false, true);
    const uint32_t q_base = smem_u32(smem + Cfg::OFF_Q);
    const uint32_t p_base = smem_u32(smem + Cfg::OFF_P);
    auto issue_s = [&](int t, int j) {  // S_t = Q_t K_j^T (caller checked kv_full)
      const int st = j % NS;
      tc_fence_after();
      const uint32_t qb = q_base + t * Cfg::Q_BYTES;
      const uint32_t kbase = smem_u32(smem + Cfg::OFF_K + st * Cfg::K_BYTES);
      if (elect_one()) {
#pragma unroll
        for (int kb = 0; kb < DH / 64; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem + t * 128, make_sw128_desc(qb + kb * (FA_BQ * 128) + k * 32, 16, 1024),
                      make_sw128_desc(kbase + kb * (FA_BK * 128) + k * 32, 16, 1024), idS, (kb | k) != 0);
        umma_commit(&s_full[t]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int t, int j) {  // O_t += P_t V_j (caller checked p_full and v_full)
      const int st = j % NSV;
      tc_fence_after();
      const uint32_t pb = p_base + t * Cfg::P_BYTES;
      const uint32_t vbase = smem_u32(smem + Cfg::OFF_V + st * Cfg::V_BYTES);
      if (elect_one()) {
#pragma unroll
        for (int kb = 0; kb < FA_BK / 64; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem + 256 + t * DH, make_sw128_desc(pb + kb * (FA_BQ * 128) + k * 32, 16, 1024),
                      make_sw128_desc(vbase + kb * (DH / 64) * 8192 + k * 2048, 8192, 1024), idO,
                      (j > 0) || ((kb | k) != 0));
        umma_commit(&o_done[t]);
      }
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    if (trc && lane == 0) trc[1] = gtime();
    const int nkt[2] = {nkt0, nkt1};
    int s_next[2] = {0, 0}, pv_next[2] = {0, 0};
    int relk = 0, relv = 0;  // next iterations whose K / V ring stage has not been released
    while (relv < n_iter) {
      bool progress = false;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int ks = s_next[t];
        // S_t(ks) may overwrite S_t(ks-1) once the group has loaded it (s_read), and needs K_ks
        if (ks < nkt[t] && (ks == 0 || mbar_test(&s_read[t], (ks - 1) & 1)) &&
            mbar_test(&kv_full[ks % NS], (ks / NS) & 1)) {
          issue_s(t, ks);
          s_next[t] = ks + 1;
          progress = true;
        }
        const int kp = pv_next[t];
        if (kp < s_next[t] && mbar_test(&p_full[t], kp & 1) && mbar_test(&v_full[kp % NSV], (kp / NSV) & 1)) {
          issue_pv(t, kp);
          pv_next[t] = kp + 1;
          progress = true;
        }
      }
      // K of iteration relk is free once every query tile using it issued its S; V once P.V
      // (a commit tracks all MMAs issued before it)
      while (relk < n_iter && (relk >= nkt0 || s_next[0] > relk) && (relk >= nkt1 || s_next[1] > relk)) {
        if (elect_one()) umma_commit(&kv_empty[relk % NS]);
        __syncwarp();
        ++relk;
        progress = true;
      }
      while (relv < n_iter && (relv >= nkt0 || pv_next[0] > relv) && (relv >= nkt1 || pv_next[1] > relv)) {
        if (elect_one()) umma_commit(&v_empty[relv % NSV]);
        __syncwarp();
        ++relv;
        progress = true;
      }
      if (!progress) __nanosleep(20);
    }
  } else if (warp >= 4) {
    // ---------------- softmax groups (thread = query row) ----------------
    const int t = (warp - 4) >> 2;  // query tile of this group
    const int nkt = t == 0 ? nkt0 : nkt1;
    const int r = (warp & 3) * 32 + lane;  // row within tile == TMEM lane
    const int qt = qt0 + t;
    const int q = qt * FA_BQ + r;
    const uint32_t t_lane = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + t * 128 + t_lane;
    const uint32_t tO = tmem + 256 + t * DH + t_lane;
    const float* mrow = a.mask ? a.mask + (int64_t)b * a.s : nullptr;
    const uint32_t* krow = a.keep ? a.keep + (((int64_t)b * a.nh + h) * a.s + q) * (a.s / 32) : nullptr;
    uint8_t* p_smem = smem + Cfg::OFF_P + t * Cfg::P_BYTES;
    // m: the running max the exponents are taken against (log2 domain).  It is only moved when
    // a row's max grows by more than 8 (P <= 2^8 stays exact enough in bf16 / fp32), so the O
    // rescale in TMEM is rare; l is kept consistent with m.
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nkt; ++j) {
      const int key0 = j * FA_BK;
      const bool diag = a.causal && (j == qt);
      uint4 kw = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
      if (krow) kw = __ldg(reinterpret_cast<const uint4*>(krow + key0 / 32));
      mbar_wait(&s_full[t], j & 1);
      if (trc && threadIdx.x == 128 && j < 8) trc[2 + j] = gtime();
      tc_fence_after();
      uint32_t sv[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sv + c * 32));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_read[t]);  // S_t may now be overwritten by S_t(j+1)
      // x = log2-domain logits; without a mask the scale is folded into the exponent's FFMA
      float* x = reinterpret_cast<float*>(sv);
      float xs = a.scale_log2;
      if (mrow) {
        const float4* mp = reinterpret_cast<const float4*>(mrow + key0);
        const float2 sl2 = make_float2(a.scale_log2, a.scale_log2);
        const float2 l2e = make_float2(1.4426950408889634f, 1.4426950408889634f);
#pragma unroll
        for (int k4 = 0; k4 < 32; ++k4) {
          const float4 mk = __ldg(mp + k4);
          const float2 y0 = __ffma2_rn(make_float2(x[4 * k4 + 0], x[4 * k4 + 1]), sl2,
                                       __fmul2_rn(make_float2(mk.x, mk.y), l2e));
          const float2 y1 = __ffma2_rn(make_float2(x[4 * k4 + 2], x[4 * k4 + 3]), sl2,
                                       __fmul2_rn(make_float2(mk.z, mk.w), l2e));
          x[4 * k4 + 0] = y0.x;
          x[4 * k4 + 1] = y0.y;
          x[4 * k4 + 2] = y1.x;
          x[4 * k4 + 3] = y1.y;
        }
        xs = 1.f;
      }
      if (diag) {
#pragma unroll
        for (int k = 0; k < 128; ++k)
          if (k > r) x[k] = -INFINITY;
      }
      float mx8[8];  // 3-input max (FMNMX3): two keys per instruction
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = x[i];
#pragma unroll
      for (int k = 8; k < 128; k += 16)
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = fmaxf(fmaxf(mx8[i], x[k + i]), x[k + 8 + i]);
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * xs;
      float alpha = 1.f;
      if (mx > m + 8.f) {  // (also the first finite max: m = -inf)
        alpha = (m == -INFINITY) ? 0.f : ex2_approx(m - mx);
        m = mx;
      }
      const float m_use = (m == -INFINITY) ? 0.f : m;
      const float nm = -m_use;
      // P = exp2(x*xs - m); row sum before dropout; dropped entries zero (1/(1-p) in the epilogue)
      // paired fp32 math (FFMA2 / FADD2) and packed keep masks: the pass is issue-bound
      uint32_t pk[64];
      float2 rs2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const uint32_t kws[4] = {kw.x, kw.y, kw.z, kw.w};
      const float2 xs2 = make_float2(xs, xs), nm2 = make_float2(nm, nm);
      uint32_t ksh[8];
#pragma unroll
      for (int k = 0; k < 128; k += 2) {
        if ((k & 31) == 0) keep_shifts(kws[k >> 5], ksh);
        const float2 y = __ffma2_rn(make_float2(x[k], x[k + 1]), xs2, nm2);
        const float2 pv = make_float2(ex2_approx(y.x), ex2_approx(y.y));
        rs2[(k >> 1) & 3] = __fadd2_rn(rs2[(k >> 1) & 3], pv);
        pk[k >> 1] = pack_bf16x2(pv.x, pv.y) & keep_pair_mask(ksh, (k & 31) >> 3, k & 7);
      }
      const float rowsum = ((rs2[0].x + rs2[0].y) + (rs2[1].x + rs2[1].y)) + ((rs2[2].x + rs2[2].y) + (rs2[3].x + rs2[3].y));
      l = l * alpha + rowsum;
      if (j > 0) {
        // P.V of tile j-1 must have finished: it reads the P buffer we overwrite below and
        // accumulates into the O we rescale
        mbar_wait(&o_done[t], (j - 1) & 1);
        tc_fence_after();
        if (!__all_sync(0xffffffffu, alpha == 1.f)) {
#pragma unroll
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st_32x32b_x32(tO + c * 32, o);
          }
          tmem_st_wait();
        }
      }
      // P -> smem as the swizzled K-major A operand (keys [64kb, 64kb+64) in sub-tile kb;
      // 16-B granule g = keys 8g..8g+7)
#pragma unroll
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const int w0 = kb * 32 + g * 4;
          *reinterpret_cast<uint4*>(p_smem + kb * (FA_BQ * 128) + sw128_offset(r, g)) =
              make_uint4(pk[w0], pk[w0 + 1], pk[w0 + 2], pk[w0 + 3]);
        }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
      if (trc && threadIdx.x == 128 && j < 8) trc[10 + j] = gtime();
    }
    // epilogue: O * (1/(1-p)) / l -> bf16; lse
    if (nkt > 0) {
      mbar_wait(&o_done[t], (nkt - 1) & 1);
      tc_fence_after();
      const float sc = l > 0.f ? a.inv_keep / l : 0.f;
      bf16* orow = a.out + ((int64_t)b * a.s + q) * a.ld_out + (int64_t)h * DH;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tO + c * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint4 u;
          u.x = pack_bf16x2(__uint_as_float(o[g * 8 + 0]) * sc, __uint_as_float(o[g * 8 + 1]) * sc);
          u.y = pack_bf16x2(__uint_as_float(o[g * 8 + 2]) * sc, __uint_as_float(o[g * 8 + 3]) * sc);
          u.z = pack_bf16x2(__uint_as_float(o[g * 8 + 4]) * sc, __uint_as_float(o[g * 8 + 5]) * sc);
          u.w = pack_bf16x2(__uint_as_float(o[g * 8 + 6]) * sc, __uint_as_float(o[g * 8 + 7]) * sc);
          *reinterpret_cast<uint4*>(orow + c * 32 + g * 8) = u;
        }
      }
      // +inf marks a fully masked row (the backward then recomputes P = exp2(... - lse) = 0)
      if (a.lse) a.lse[((int64_t)b * a.nh + h) * a.s + q] = (l > 0.f) ? m + __log2f(l) : INFINITY;
      if (trc && threadIdx.x == 128) trc[18] = gtime();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, Cfg::TMEM_COLS);
  }
}

// Attention-probability dropout keep bits (site 0 of the Philox scheme, oracle/philox.py):
// word ((b*nh + h)*sq + q)*(sk/32) + k/32, bit k%32 = keep(row = (gs*nh_global + gh)*sq + q,
// col = k) with gs = sample_offset + (b / sample_block) * block_stride + b % sample_block (blocks of
// sample_block consecutive samples block_stride apart: an overlapped micro-batch's rank-major
// gathered samples), gh = head_offset + h.  One thread per word
// (4 Philox4x32-10 calls = 32 keys).
__global__ void __launch_bounds__(128) attn_dropout_bits_kernel(int nh, int sq, int wpr, uint32_t thresh,
                                                                uint64_t seed, const uint64_t* rng_step,
                                                                uint32_t layer,
                                                                int64_t sample_offset, int sample_block,
                                                                int64_t block_stride, int head_offset, int nh_global,
                                                                uint32_t* __restrict__ bits, int causal) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // (q, w) of this (b, h)
  if (idx >= sq * wpr) return;
  // causal: the kernels never read words of key tiles after the query's tile (128-key tiles)
  if (causal && ((idx % wpr) >> 2) > (idx / wpr) >> 7) return;
  const uint64_t pkey = philox_key(seed, rng_step);
  const PhiloxRoundKeys rk = philox_round_keys(static_cast<uint32_t>(pkey), static_cast<uint32_t>(pkey >> 32));
  const int bh = blockIdx.y;
  const int q = idx / wpr, w = idx - q * wpr;
  const int h = bh % nh, b = bh / nh;
  const int64_t gs = sample_offset + (int64_t)(b / sample_block) * block_stride + b % sample_block;
  const uint64_t grow = (uint64_t)((gs * nh_global + head_offset + h) * (int64_t)sq + q);
  uint32_t word = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) word |= dropout_keep8_bits(rk, layer, 0u, grow, w * 32 + c * 8, thresh) << (c * 8);
  bits[(int64_t)bh * sq * wpr + idx] = word;
}

}  // namespace smpk

using namespace smpk;

extern "C" int smpk_attn_dropout_bits_blocked(int B, int nh, int sq, int sk, float p_drop, uint64_t seed,
                                              const uint64_t* rng_step, int layer, int64_t sample_offset,
                                              int sample_block, int64_t block_stride, int head_offset, int nh_global,
                                              uint32_t* bits, int causal, void* stream) {
  SMPK_REQUIRE(B > 0 && nh > 0 && sq > 0 && sk > 0 && sk % 32 == 0 && bits, SMPK_ERR_BAD_ARG,
               "smpk_attn_dropout_bits: bad arguments (sk must be a multiple of 32)");
  SMPK_REQUIRE(p_drop >= 0.f && p_drop < 1.f, SMPK_ERR_BAD_ARG, "smpk_attn_dropout_bits: p in [0,1)");
  SMPK_REQUIRE((int64_t)B * nh < 65536, SMPK_ERR_UNSUPPORTED, "smpk_attn_dropout_bits: B*nh must be < 65536");
  SMPK_REQUIRE(sample_block > 0, SMPK_ERR_BAD_ARG, "smpk_attn_dropout_bits: sample_block must be > 0");
  const int wpr = sk / 32;
  dim3 grid((unsigned)((sq * wpr + 127) / 128), (unsigned)(B * nh));
  attn_dropout_bits_kernel<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      nh, sq, wpr, dropout_threshold(p_drop), seed, rng_step, (uint32_t)layer, sample_offset, sample_block,
      block_stride, head_offset, nh_global, bits, causal);
  return check_launch("smpk_attn_dropout_bits");
}

extern "C" int smpk_attn_dropout_bits(int B, int nh, int sq, int sk, float p_drop, uint64_t seed,
                                      const uint64_t* rng_step, int layer,
                                      int64_t sample_offset, int head_offset, int nh_global, uint32_t* bits,
                                      int causal, void* stream) {
  return smpk_attn_dropout_bits_blocked(B, nh, sq, sk, p_drop, seed, rng_step, layer, sample_offset, B > 0 ? B : 1, 0,
                                        head_offset, nh_global, bits, causal, stream);
}

extern "C" int smpk_flash_attn_fwd(const void* qkv, int64_t ld, int B, int nh, int s, int dh, void* out,
                                   int64_t ld_out, float* lse, const float* mask_add, float scale, int causal,
                                   float p_drop, const uint32_t* keep_bits, void* stream) {
  SMPK_REQUIRE(dh == 64 || dh == 128, SMPK_ERR_UNSUPPORTED, "smpk_flash_attn_fwd: head dim %d (64 or 128)", dh);
  SMPK_REQUIRE(s % 128 == 0 && s > 0, SMPK_ERR_UNSUPPORTED, "smpk_flash_attn_fwd: seq %d must be a multiple of 128",
               s);
  SMPK_REQUIRE(qkv && out && B > 0 && nh > 0, SMPK_ERR_BAD_ARG, "smpk_flash_attn_fwd: bad arguments");
  SMPK_REQUIRE(p_drop >= 0.f && p_drop < 1.f, SMPK_ERR_BAD_ARG, "smpk_flash_attn_fwd: dropout p in [0,1)");
  SMPK_REQUIRE(p_drop == 0.f || keep_bits, SMPK_ERR_BAD_ARG, "smpk_flash_attn_fwd: dropout needs keep bits");
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
  a.keep = p_drop > 0.f ? keep_bits : nullptr;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.causal = causal;
  a.inv_keep = p_drop > 0.f ? 1.f / (1.f - p_drop) : 1.f;
  static int trace_env = -1;
  if (trace_env < 0) {
    const char* e = getenv("SMPK_FA_TRACE");
    trace_env = (e && e[0] == '1') ? 1 : 0;
  }
  a.trace = trace_env;
  dim3 grid((s / 128 + 1) / 2, nh, B);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dh == 64) {
    static unsigned long long once = 0;
    smem_attr_once(flash_fwd_kernel<64, 3, 3>, FaFwdCfg<64, 3, 3>::SMEM, once);
    launch_pdl(flash_fwd_kernel<64, 3, 3>, grid, FA_THREADS, FaFwdCfg<64, 3, 3>::SMEM, st, tq, tk, tv, a);
  } else {
    static unsigned long long once = 0;
    smem_attr_once(flash_fwd_kernel<128, 2, 1>, FaFwdCfg<128, 2, 1>::SMEM, once);
    launch_pdl(flash_fwd_kernel<128, 2, 1>, grid, FA_THREADS, FaFwdCfg<128, 2, 1>::SMEM, st, tq, tk, tv, a);
  }
  return check_launch("smpk_flash_attn_fwd");
}

// debug: copy the forward timeline records of the last traced launch (SMPK_FA_TRACE=1)
extern "C" int smpk_debug_fa_trace(void* host_out, int n_cta) {
  if (n_cta > 1024) n_cta = 1024;
  cudaError_t e = cudaMemcpyFromSymbol(host_out, smpk::g_fa_trace, (size_t)n_cta * 20 * 8);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_debug_fa_trace: %s", cudaGetErrorString(e));
  return SMPK_OK;
}

// gemm.cu — warp-specialised persistent tcgen05 GEMM for sm_100a.
//
// One CTA per SM.  Warp 0 lane 0 drives TMA (4-D tensor maps, SWIZZLE_128B) into
// a STAGES-deep smem ring; warp 1 lane 0 issues tcgen05.mma (M=128, N=BN, K=16)
// into a double-buffered TMEM accumulator; warps 4..7 drain TMEM with
// tcgen05.ld, apply the fused epilogue (bias / activation / activation-backward
// / residual / beta-accumulate) and store to HBM, overlapping the next tile's
// main loop.  Both operand majors are supported through the UMMA descriptor, so
// forward, dgrad and wgrad of every linear map onto the same kernel without
// transposes.
//
// Hot-path role: the local GEMM of DistributedLinear / column- and row-parallel
// transformer linears and the per-head
// attention contractions.
#include <cstdarg>
#include <cstdio>
#include <mutex>

#include "smpk_common.cuh"

namespace smpk {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int GEMM_THREADS = 384;  // warps 0-3: TMA, MMA, TMEM alloc, spare; 4-11: epilogue

struct GemmArgs {
  int M, N, K;
  int nb1, nb2;
  int tiles_m, tiles_n, num_tiles, num_kb;
  int a_mn, b_mn;
  void* c;
  int c_f32;
  int64_t ldc, c_bs1, c_bs2;
  float alpha, beta;
  int epi, act;
  const bf16* bias;
  bf16* aux;
  int64_t ldaux;
  int vec_ok;  // 16B-aligned rows of C / aux
  // reduce-scatter epilogue: row r of C goes to rank (r / rows_per_owner)'s peer-mapped
  // buffer c_peers[owner] at element offset peer_slot_off + (r % rows_per_owner) * ldc
  void* const* c_peers;
  int64_t rows_per_owner, peer_slot_off;
};

template <int BN, int STAGES>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256 /*barriers*/;
};

__device__ __forceinline__ void decode_tile(const GemmArgs& g, int tile, int& b1, int& b2, int& tm, int& tn) {
  int per = g.tiles_m * g.tiles_n;
  int b = tile / per;
  int r = tile - b * per;
  tn = r / g.tiles_m;
  tm = r - tn * g.tiles_m;
  b1 = b % g.nb1;
  b2 = b / g.nb1;
}

// Epilogue for 32 consecutive accumulator columns of one row.  EPI / ACT / F32OUT /
// BETA are compile-time so every instantiation is a straight-line, branch-free body.
template <int EPI, int ACT, bool F32OUT, bool BETA>
__device__ __forceinline__ void epilogue_store32(const GemmArgs& g, int row, int col0, int64_t c_off,
                                                 const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * g.alpha;
  const bool full = (col0 + 32 <= g.N) && g.vec_ok;

  if constexpr (EPI == SMPK_EPI_BIAS || EPI == SMPK_EPI_BIAS_ACT) {
    if (full) {
      const uint4* bp = reinterpret_cast<const uint4*>(g.bias + col0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u = __ldg(bp + q);
        uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 f = unpack_bf16x2(w[j]);
          v[q * 8 + 2 * j] += f.x;
          v[q * 8 + 2 * j + 1] += f.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) v[i] += bf2f(g.bias[col0 + i]);
    }
  }

  if constexpr (EPI == SMPK_EPI_BIAS_ACT || EPI == SMPK_EPI_DACT || EPI == SMPK_EPI_ADD) {
    bf16* ap = g.aux + c_off + (int64_t)row * g.ldaux + col0;
    if constexpr (EPI == SMPK_EPI_BIAS_ACT) {
      // store the pre-activation, then activate its bf16 rounding (what backward re-reads)
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = round_bf16(v[i]);
      if (full) {
        uint4* d = reinterpret_cast<uint4*>(ap);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          u.x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
          u.y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
          u.z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
          u.w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
          d[q] = u;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < g.N) ap[i] = f2bf(v[i]);
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = act_fwd(ACT, v[i]);
    } else {
      float a[32];
      if (full) {
        const uint4* src = reinterpret_cast<const uint4*>(ap);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u = src[q];
          uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float2 f = unpack_bf16x2(w[j]);
            a[q * 8 + 2 * j] = f.x;
            a[q * 8 + 2 * j + 1] = f.y;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) a[i] = (col0 + i < g.N) ? bf2f(ap[i]) : 0.f;
      }
      if constexpr (EPI == SMPK_EPI_DACT) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= act_bwd(ACT, a[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += a[i];
      }
    }
  }

  if constexpr (F32OUT) {
    float* cp = reinterpret_cast<float*>(g.c) + c_off + (int64_t)row * g.ldc + col0;
    if (full) {
      float4* d = reinterpret_cast<float4*>(cp);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        if constexpr (BETA) {
          float4 old = d[q];
          o.x += g.beta * old.x;
          o.y += g.beta * old.y;
          o.z += g.beta * old.z;
          o.w += g.beta * old.w;
        }
        d[q] = o;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) cp[i] = v[i] + (BETA ? g.beta * cp[i] : 0.f);
    }
  } else {
    bf16* cp;
    if (g.c_peers != nullptr) {  // NVLink peer store into the owning rank's partial slot
      const int64_t owner = row / g.rows_per_owner;
      cp = reinterpret_cast<bf16*>(g.c_peers[owner]) + g.peer_slot_off + (row - owner * g.rows_per_owner) * g.ldc +
           col0;
    } else {
      cp = reinterpret_cast<bf16*>(g.c) + c_off + (int64_t)row * g.ldc + col0;
    }
    if (full) {
      uint4* d = reinterpret_cast<uint4*>(cp);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if constexpr (BETA) {
          uint4 old = d[q];
          uint32_t w[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float2 f = unpack_bf16x2(w[j]);
            v[q * 8 + 2 * j] += g.beta * f.x;
            v[q * 8 + 2 * j + 1] += g.beta * f.y;
          }
        }
        uint4 u;
        u.x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
        u.y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
        u.z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
        u.w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
        d[q] = u;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) cp[i] = f2bf(v[i] + (BETA ? g.beta * bf2f(cp[i]) : 0.f));
    }
  }
}

template <int BN, int STAGES, int EPI, int ACT, bool F32OUT, bool BETA>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const GemmArgs g) {
  using Cfg = GemmCfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::B_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 256);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x) {
        int b1, b2, tm, tn;
        decode_tile(g, tile, b1, b2, tm, tn);
        for (int kb = 0; kb < g.num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          uint8_t* a_dst = sA + stage * Cfg::A_BYTES;
          uint8_t* b_dst = sB + stage * Cfg::B_BYTES;
          if (!g.a_mn) {
            tma_load_4d(a_dst, &tmA, &full_bar[stage], kb * BK, tm * BM, b1, b2);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              tma_load_4d(a_dst + i * (BK * 128), &tmA, &full_bar[stage], tm * BM + i * 64, kb * BK, b1, b2);
          }
          if (!g.b_mn) {
            tma_load_4d(b_dst, &tmB, &full_bar[stage], kb * BK, tn * BN, b1, b2);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_4d(b_dst + i * (BK * 128), &tmB, &full_bar[stage], tn * BN + i * 64, kb * BK, b1, b2);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t idesc = make_idesc_bf16(BM, BN, g.a_mn, g.b_mn);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < g.num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t adesc = g.a_mn ? make_sw128_desc(a_base + k * 2048, BK * 128, 1024)
                                          : make_sw128_desc(a_base + k * 32, 16, 1024);
            const uint64_t bdesc = g.b_mn ? make_sw128_desc(b_base + k * 2048, BK * 128, 1024)
                                          : make_sw128_desc(b_base + k * 32, 16, 1024);
            umma_bf16(d_tmem, adesc, bdesc, idesc, (kb | k) != 0);
          }
          umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull_bar[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    // 8 warps: warp%4 selects the TMEM lane quarter (hardware rule), (warp-4)/4 the column half
    const int quarter = warp & 3;
    const int half = (warp - 4) >> 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x) {
      int b1, b2, tm, tn;
      decode_tile(g, tile, b1, b2, tm, tn);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = tm * BM + quarter * 32 + lane;
      const int64_t c_off = (int64_t)b1 * g.c_bs1 + (int64_t)b2 * g.c_bs2;
      const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16);
      // software-pipelined TMEM drain: the load of chunk i+1 is in flight while chunk i
      // is processed and stored (tcgen05.wait::ld waits for all earlier loads).
      constexpr int CH = BN / 64;  // 32-column chunks per warp
      const int c_first = half * CH;
      uint32_t r[2][32];
      tmem_ld_32x32b_x32(t_row + c_first * 32, r[0]);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        if (i + 1 < CH) tmem_ld_32x32b_x32(t_row + (c_first + i + 1) * 32, r[(i + 1) & 1]);
        const int col0 = tn * BN + (c_first + i) * 32;
        if (row < g.M && col0 < g.N) epilogue_store32<EPI, ACT, F32OUT, BETA>(g, row, col0, c_off, r[i & 1]);
        if (i + 1 < CH) tmem_ld_wait();
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                      CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  return fn;
}

// 4-D bf16 tensor map {inner, outer, nb1, nb2} with SWIZZLE_128B boxes {box_inner, box_outer, 1, 1}.
int make_tma_4d(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int nb1, int64_t s1,
                int nb2, int64_t s2, int box_inner, int box_outer, const char* name) {
  PFN_encodeTiled_t enc = get_encode_fn();
  SMPK_REQUIRE(enc != nullptr, SMPK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  SMPK_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, SMPK_ERR_BAD_ARG,
               "operand %s must be 16-byte aligned", name);
  SMPK_REQUIRE(ld % 8 == 0, SMPK_ERR_BAD_ARG, "leading dim of %s (%lld) must be a multiple of 8", name,
               (long long)ld);
  SMPK_REQUIRE((nb1 == 1 || s1 % 8 == 0) && (nb2 == 1 || s2 % 8 == 0), SMPK_ERR_BAD_ARG,
               "batch strides of %s must be multiples of 8", name);
  cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)nb1, (cuuint64_t)nb2};
  const int64_t fallback = ld * outer * 2;
  cuuint64_t strides[3] = {(cuuint64_t)(ld * 2), (cuuint64_t)(nb1 > 1 ? s1 * 2 : fallback),
                           (cuuint64_t)(nb2 > 1 ? s2 * 2 : fallback)};
  cuuint32_t box[4] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer, 1u, 1u};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SMPK_REQUIRE(r == CUDA_SUCCESS, SMPK_ERR_CUDA, "tensor map for %s failed (CUresult %d)", name, (int)r);
  return SMPK_OK;
}

// Operand view: rows x K logical, either K-major (K contiguous) or MN-major.
static int make_operand_map(CUtensorMap* map, const void* ptr, bool mn_major, int rows, int K, int64_t ld,
                            int nb1, int64_t s1, int nb2, int64_t s2, int box_rows, const char* name) {
  return make_tma_4d(map, ptr, mn_major ? rows : K, mn_major ? K : rows, ld, nb1, s1, nb2, s2, 64,
                     mn_major ? BK : box_rows, name);
}

template <int BN, int STAGES, int EPI, int ACT, bool F32OUT, bool BETA>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, GemmArgs& g, cudaStream_t st) {
  using Cfg = GemmCfg<BN, STAGES>;
  auto kern = gemm_bf16_tcgen05<BN, STAGES, EPI, ACT, F32OUT, BETA>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_gemm: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  g.tiles_n = (g.N + BN - 1) / BN;
  g.num_tiles = g.tiles_m * g.tiles_n * g.nb1 * g.nb2;
  int grid = g.num_tiles < num_sms() ? g.num_tiles : num_sms();
  kern<<<grid, GEMM_THREADS, Cfg::SMEM_BYTES, st>>>(ta, tb, g);
  return check_launch("smpk_gemm");
}

template <int BN, int STAGES>
static int dispatch_epilogue(const CUtensorMap& ta, const CUtensorMap& tb, GemmArgs& g, cudaStream_t st) {
  const bool beta = g.beta != 0.f;
  switch (g.epi) {
    case SMPK_EPI_NONE:
      if (g.c_f32) return beta ? launch_gemm<BN, STAGES, SMPK_EPI_NONE, 0, true, true>(ta, tb, g, st)
                               : launch_gemm<BN, STAGES, SMPK_EPI_NONE, 0, true, false>(ta, tb, g, st);
      return beta ? launch_gemm<BN, STAGES, SMPK_EPI_NONE, 0, false, true>(ta, tb, g, st)
                  : launch_gemm<BN, STAGES, SMPK_EPI_NONE, 0, false, false>(ta, tb, g, st);
    case SMPK_EPI_BIAS:
      if (g.c_f32 || beta) break;
      return launch_gemm<BN, STAGES, SMPK_EPI_BIAS, 0, false, false>(ta, tb, g, st);
    case SMPK_EPI_BIAS_ACT:
      if (g.c_f32 || beta) break;
      if (g.act == SMPK_ACT_GELU_ERF) return launch_gemm<BN, STAGES, SMPK_EPI_BIAS_ACT, SMPK_ACT_GELU_ERF, false, false>(ta, tb, g, st);
      if (g.act == SMPK_ACT_GELU_TANH) return launch_gemm<BN, STAGES, SMPK_EPI_BIAS_ACT, SMPK_ACT_GELU_TANH, false, false>(ta, tb, g, st);
      if (g.act == SMPK_ACT_RELU) return launch_gemm<BN, STAGES, SMPK_EPI_BIAS_ACT, SMPK_ACT_RELU, false, false>(ta, tb, g, st);
      break;
    case SMPK_EPI_DACT:
      if (g.c_f32 || beta) break;
      if (g.act == SMPK_ACT_GELU_ERF) return launch_gemm<BN, STAGES, SMPK_EPI_DACT, SMPK_ACT_GELU_ERF, false, false>(ta, tb, g, st);
      if (g.act == SMPK_ACT_GELU_TANH) return launch_gemm<BN, STAGES, SMPK_EPI_DACT, SMPK_ACT_GELU_TANH, false, false>(ta, tb, g, st);
      if (g.act == SMPK_ACT_RELU) return launch_gemm<BN, STAGES, SMPK_EPI_DACT, SMPK_ACT_RELU, false, false>(ta, tb, g, st);
      break;
    case SMPK_EPI_ADD:
      if (g.c_f32 || beta) break;
      return launch_gemm<BN, STAGES, SMPK_EPI_ADD, 0, false, false>(ta, tb, g, st);
  }
  set_last_error("smpk_gemm: unsupported epilogue combination epi=%d act=%d c_f32=%d beta=%g", g.epi, g.act, g.c_f32,
                 g.beta);
  return SMPK_ERR_UNSUPPORTED;
}

}  // namespace smpk

using namespace smpk;

static int gemm_impl(const void* a, int a_mn_major, int64_t lda, int64_t a_bs1, int64_t a_bs2, const void* b,
                     int b_mn_major, int64_t ldb, int64_t b_bs1, int64_t b_bs2, void* c, int c_f32, int64_t ldc,
                     int64_t c_bs1, int64_t c_bs2, int M, int N, int K, int nb1, int nb2, float alpha, float beta,
                     int epilogue, int act, const void* bias, void* aux, int64_t ldaux, void* const* c_peers,
                     int64_t rows_per_owner, int64_t peer_slot_off, void* stream) {
  SMPK_REQUIRE(M > 0 && N > 0 && K > 0 && nb1 > 0 && nb2 > 0, SMPK_ERR_BAD_SHAPE,
               "smpk_gemm: bad shape M=%d N=%d K=%d nb=%dx%d", M, N, K, nb1, nb2);
  SMPK_REQUIRE(a && b && (c || c_peers), SMPK_ERR_BAD_ARG, "smpk_gemm: null operand");
  SMPK_REQUIRE(epilogue >= SMPK_EPI_NONE && epilogue <= SMPK_EPI_ADD, SMPK_ERR_BAD_ARG,
               "smpk_gemm: unknown epilogue %d", epilogue);
  const bool need_bias = epilogue == SMPK_EPI_BIAS || epilogue == SMPK_EPI_BIAS_ACT;
  const bool need_aux = epilogue == SMPK_EPI_BIAS_ACT || epilogue == SMPK_EPI_DACT || epilogue == SMPK_EPI_ADD;
  SMPK_REQUIRE(!need_bias || bias, SMPK_ERR_BAD_ARG, "smpk_gemm: epilogue %d needs bias", epilogue);
  SMPK_REQUIRE(!need_aux || aux, SMPK_ERR_BAD_ARG, "smpk_gemm: epilogue %d needs aux", epilogue);
  SMPK_REQUIRE(!(need_aux && c_f32), SMPK_ERR_UNSUPPORTED, "smpk_gemm: aux epilogues need bf16 C");

  int BN = N <= 64 ? 64 : (N <= 128 ? 128 : 256);

  CUtensorMap ta, tb;
  int rc = make_operand_map(&ta, a, a_mn_major, M, K, lda, nb1, a_bs1, nb2, a_bs2, BM, "A");
  if (rc) return rc;
  rc = make_operand_map(&tb, b, b_mn_major, N, K, ldb, nb1, b_bs1, nb2, b_bs2, BN, "B");
  if (rc) return rc;

  GemmArgs g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.nb1 = nb1;
  g.nb2 = nb2;
  g.tiles_m = (M + BM - 1) / BM;
  g.num_kb = (K + BK - 1) / BK;
  g.a_mn = a_mn_major ? 1 : 0;
  g.b_mn = b_mn_major ? 1 : 0;
  g.c = c;
  g.c_f32 = c_f32 ? 1 : 0;
  g.ldc = ldc;
  g.c_bs1 = c_bs1;
  g.c_bs2 = c_bs2;
  g.alpha = alpha;
  g.beta = beta;
  g.epi = epilogue;
  g.act = act;
  g.bias = reinterpret_cast<const bf16*>(bias);
  g.aux = reinterpret_cast<bf16*>(aux);
  g.ldaux = ldaux;
  g.c_peers = c_peers;
  g.rows_per_owner = rows_per_owner > 0 ? rows_per_owner : 1;
  g.peer_slot_off = peer_slot_off;
  const int esz = c_f32 ? 4 : 2;
  bool vec = (reinterpret_cast<uintptr_t>(c) % 16 == 0) && ((ldc * esz) % 16 == 0) && ((c_bs1 * esz) % 16 == 0) &&
             ((c_bs2 * esz) % 16 == 0);
  if (c_peers) vec = ((ldc * esz) % 16 == 0) && ((peer_slot_off * esz) % 16 == 0);
  if (need_bias) vec = vec && (reinterpret_cast<uintptr_t>(bias) % 16 == 0);
  if (need_aux) vec = vec && (reinterpret_cast<uintptr_t>(aux) % 16 == 0) && (ldaux % 8 == 0);
  g.vec_ok = vec ? 1 : 0;

  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (BN == 64) return dispatch_epilogue<64, 8>(ta, tb, g, st);
  if (BN == 128) return dispatch_epilogue<128, 6>(ta, tb, g, st);
  return dispatch_epilogue<256, 4>(ta, tb, g, st);
}

extern "C" int smpk_gemm(const void* a, int a_mn_major, int64_t lda, int64_t a_bs1, int64_t a_bs2, const void* b,
                         int b_mn_major, int64_t ldb, int64_t b_bs1, int64_t b_bs2, void* c, int c_f32,
                         int64_t ldc, int64_t c_bs1, int64_t c_bs2, int M, int N, int K, int nb1, int nb2,
                         float alpha, float beta, int epilogue, int act, const void* bias, void* aux,
                         int64_t ldaux, void* stream) {
  return gemm_impl(a, a_mn_major, lda, a_bs1, a_bs2, b, b_mn_major, ldb, b_bs1, b_bs2, c, c_f32, ldc, c_bs1, c_bs2,
                   M, N, K, nb1, nb2, alpha, beta, epilogue, act, bias, aux, ldaux, nullptr, 0, 0, stream);
}

extern "C" int smpk_gemm_rs(const void* a, int a_mn_major, int64_t lda, const void* b, int b_mn_major, int64_t ldb,
                            void* const* c_peers, int64_t ldc, int64_t rows_per_owner, int64_t peer_slot_off, int M,
                            int N, int K, void* stream) {
  SMPK_REQUIRE(c_peers != nullptr, SMPK_ERR_BAD_ARG, "smpk_gemm_rs: null peer table");
  SMPK_REQUIRE(rows_per_owner > 0 && rows_per_owner % 128 == 0 && M % rows_per_owner == 0, SMPK_ERR_NOT_DIVISIBLE,
               "smpk_gemm_rs: rows per owner %lld must divide M=%d and be a multiple of 128",
               (long long)rows_per_owner, M);
  return gemm_impl(a, a_mn_major, lda, 0, 0, b, b_mn_major, ldb, 0, 0, nullptr, 0, ldc, 0, 0, M, N, K, 1, 1, 1.f,
                   0.f, SMPK_EPI_NONE, 0, nullptr, nullptr, 0, c_peers, rows_per_owner, peer_slot_off, stream);
}

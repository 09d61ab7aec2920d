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
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "smpk_common.cuh"

namespace smpk {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row

// Epilogue warps (warps 4..): 16 for the activation epilogues (issue-heavy: GeLU / dGeLU per
// element), 8 otherwise — fewer staging boxes leave room for a deeper operand ring.
__host__ __device__ constexpr int epi_warps(int epi) {
  return (epi == SMPK_EPI_BIAS_ACT || epi == SMPK_EPI_DACT) ? 16 : 8;
}
__host__ __device__ constexpr int gemm_threads(int epi) { return 128 + 32 * epi_warps(epi); }
constexpr int STG_BYTES = 4096;                             // TMA-store staging per epilogue warp
constexpr int MAX_PEERS = 8;

struct GemmArgs {
  int M, N, K;
  int nb1, nb2;
  int tiles_m, tiles_n, num_tiles, num_kb;
  int a_mn, b_mn;
  // batch dims in which an operand is broadcast (batch stride 0): its TMA coordinate stays 0
  int a_bc1, a_bc2, b_bc1, b_bc2;
  void* c;
  int c_f32;
  int64_t ldc, c_bs1, c_bs2;
  float alpha, beta;
  int epi, act;
  const bf16* bias;
  bf16* aux;
  int64_t ldaux;
  int vec_ok;     // 16B-aligned rows of C / aux (direct-store fallback)
  int tma_store;  // C (and the BIAS_ACT pre-activation) leave through smem + TMA bulk stores
  // reduce-scatter epilogue: row r of C goes to rank (r / rows_per_owner)'s peer-mapped
  // buffer (EpiMaps::peer[owner], rows [0, rows_per_owner) of its slot)
  int npeers;
  int64_t rows_per_owner;
  // split-K: work unit u = split * num_tiles + tile covers k-blocks [split*kb_per, ...);
  // every split stores its fp32 partial tile to ws, the tile's splits then reduce it in
  // split order (deterministic) and run the epilogue.
  int splits, kb_per, num_units;
  float* ws;
  int* sem;
  // fused bias-gradient column sums (TMA-store path): colsum_part[row / 32][col] = sum of the 32
  // stored bf16 rows of each output box (ceil(M/32) partial rows, reduced afterwards in order)
  float* colsum_part;
  unsigned long long* trace;  // debug timeline (SMPK_GEMM_TRACE=1), else null
};

// debug: per CTA 40 u64: [0] start, per unit k < 8: [1+4k] main loop start (MMA warp), [2+4k] last
// k-block issued, [3+4k] accumulator ready (epilogue warp 4), [4+4k] epilogue done (warp 4)
__device__ unsigned long long g_gemm_trace[2048 * 40];
__device__ __forceinline__ unsigned long long gtime_g() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// TMA store descriptors: C, the pre-activation (BIAS_ACT) and, for the reduce-scatter
// epilogue, one descriptor per owning rank's peer-mapped partial slot.
struct EpiMaps {
  CUtensorMap c;
  CUtensorMap aux;
  CUtensorMap peer[MAX_PEERS];
};

template <int BN, int STAGES, bool PAIR = false, int EPW = 8>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM_BYTES =
      1024 /*align slack*/ + STAGES * STAGE_BYTES + EPW * STG_BYTES + 256 /*barriers*/;
};

__device__ __forceinline__ void decode_unit(const GemmArgs& g, int u, int& tile, int& kb0, int& kb1) {
  const int split = u / g.num_tiles;
  tile = u - split * g.num_tiles;
  kb0 = split * g.kb_per;
  kb1 = min(kb0 + g.kb_per, g.num_kb);
}

__device__ __forceinline__ void decode_tile(const GemmArgs& g, int tile, int& b1, int& b2, int& tm, int& tn) {
  int per = g.tiles_m * g.tiles_n;
  int b = tile / per;
  int r = tile - b * per;
  tn = r / g.tiles_m;
  tm = r - tn * g.tiles_m;
  b1 = b % g.nb1;
  b2 = b / g.nb1;
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Fused epilogue math for 32 consecutive accumulator columns of one row: v = alpha * acc
// (+ bias) (-> store pre-activation, activate) (* act'(aux)) (+ aux) (+ beta * C).
// For BIAS_ACT the bf16 pre-activation is returned packed in pre[16].
template <int EPI, int ACT, bool F32OUT, bool BETA>
__device__ __forceinline__ void epilogue_math32(const GemmArgs& g, bool in_rows, int row, int col0, int64_t c_off,
                                                float (&v)[32], uint32_t (&pre)[16], const uint4* auxv = nullptr) {
  const bool full = (col0 + 32 <= g.N) && g.vec_ok;
  if (g.alpha != 1.f) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= g.alpha;
  }
  if constexpr (EPI == SMPK_EPI_BIAS || EPI == SMPK_EPI_BIAS_ACT) {
    if (full) {
      const uint4* bp = reinterpret_cast<const uint4*>(g.bias + col0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u = __ldg(bp + q);
        uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __fadd2_rn(make_float2(v[q * 8 + 2 * j], v[q * 8 + 2 * j + 1]), unpack_bf16x2(w[j]));
          v[q * 8 + 2 * j] = f.x;
          v[q * 8 + 2 * j + 1] = f.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) v[i] += bf2f(g.bias[col0 + i]);
    }
  }
  if constexpr (EPI == SMPK_EPI_BIAS_ACT) {
    // keep the pre-activation's bf16 rounding (what backward re-reads) and activate it
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      pre[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
      const float2 f = act_fwd2(ACT, unpack_bf16x2(pre[j]));
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    }
  }
  if constexpr (EPI == SMPK_EPI_DACT || EPI == SMPK_EPI_ADD) {
    if (in_rows) {
      const bf16* ap = g.aux + c_off + (int64_t)row * g.ldaux + col0;
      if (full) {
        const uint4* src = reinterpret_cast<const uint4*>(ap);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u = auxv ? auxv[q] : src[q];
          uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = unpack_bf16x2(w[j]);
            const float2 cur = make_float2(v[q * 8 + 2 * j], v[q * 8 + 2 * j + 1]);
            const float2 r = (EPI == SMPK_EPI_DACT) ? __fmul2_rn(cur, act_bwd2(ACT, f)) : __fadd2_rn(cur, f);
            v[q * 8 + 2 * j] = r.x;
            v[q * 8 + 2 * j + 1] = r.y;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float a = (col0 + i < g.N) ? bf2f(ap[i]) : 0.f;
          if constexpr (EPI == SMPK_EPI_DACT) v[i] *= act_bwd(ACT, a);
          else v[i] += a;
        }
      }
    }
  }
  if constexpr (BETA) {
    if (in_rows) {
      if constexpr (F32OUT) {
        const float* cp = reinterpret_cast<const float*>(g.c) + c_off + (int64_t)row * g.ldc + col0;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < g.N) v[i] += g.beta * cp[i];
      } else {
        const bf16* cp = reinterpret_cast<const bf16*>(g.c) + c_off + (int64_t)row * g.ldc + col0;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < g.N) v[i] += g.beta * bf2f(cp[i]);
      }
    }
  }
}

// Direct-store fallback (C rows not TMA-compatible, and the split-K fix-up).
template <int EPI, bool F32OUT>
__device__ __forceinline__ void epilogue_direct32(const GemmArgs& g, int row, int col0, int64_t c_off,
                                                  const float (&v)[32], const uint32_t (&pre)[16]) {
  const bool full = (col0 + 32 <= g.N) && g.vec_ok;
  if constexpr (EPI == SMPK_EPI_BIAS_ACT) {
    bf16* ap = g.aux + c_off + (int64_t)row * g.ldaux + col0;
    if (full) {
      uint4* d = reinterpret_cast<uint4*>(ap);
#pragma unroll
      for (int q = 0; q < 4; ++q) d[q] = make_uint4(pre[4 * q], pre[4 * q + 1], pre[4 * q + 2], pre[4 * q + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) {
          const float2 f = unpack_bf16x2(pre[i >> 1]);
          ap[i] = f2bf((i & 1) ? f.y : f.x);
        }
    }
  }
  if constexpr (F32OUT) {
    float* cp = reinterpret_cast<float*>(g.c) + c_off + (int64_t)row * g.ldc + col0;
    if (full) {
      float4* d = reinterpret_cast<float4*>(cp);
#pragma unroll
      for (int q = 0; q < 8; ++q) d[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) cp[i] = v[i];
    }
  } else {
    bf16* cp = reinterpret_cast<bf16*>(g.c) + c_off + (int64_t)row * g.ldc + col0;
    if (full) {
      uint4* d = reinterpret_cast<uint4*>(cp);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        d[q] = make_uint4(pack_bf16x2(v[8 * q], v[8 * q + 1]), pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                          pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) cp[i] = f2bf(v[i]);
    }
  }
}

// Stage one lane's 32 values into the warp's swizzled TMA-store box (32 rows x 32 columns):
// bf16 -> 64-B rows, SWIZZLE_64B (16-B granule c of row r at c ^ ((r >> 1) & 3));
// fp32 -> 128-B rows, SWIZZLE_128B (granule c at c ^ (r & 7)).  8 consecutive lanes cover all
// 32 banks once, so the staging writes are conflict-free.
__device__ __forceinline__ void stage_bf16_row(uint8_t* box, int r, const uint32_t (&w)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint4* d = reinterpret_cast<uint4*>(box + r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
    *d = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
  }
}
__device__ __forceinline__ void stage_f32_row(uint8_t* box, int r, const float (&v)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    float4* d = reinterpret_cast<float4*>(box + r * 128 + ((c ^ (r & 7)) << 4));
    *d = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
}

// Kernel body.  PAIR == false: one CTA per tile of 128 x BN (tcgen05 cta_group::1).
// PAIR == true: a 2-CTA cluster on one TPC owns a 256 x BN tile; each CTA stages its 128 rows
// of A and half (BN/2 rows) of B, the leader issues M=256 cta_group::2 MMAs that read both
// CTAs' shared memory, and each CTA's TMEM receives the accumulator of its own 128 rows —
// halving the per-SM operand traffic through shared memory, the limit of the 1-CTA form.
template <int BN, int STAGES, int EPI, int ACT, bool F32OUT, bool BETA, bool PAIR, int NPROB = 1>
__device__ __forceinline__ void gemm_body(const CUtensorMap* tmA_arr, const CUtensorMap* tmB_arr,
                                          const EpiMaps* maps_arr, const GemmArgs* gs) {
  // NPROB == 2 (grouped launch): problem 1 is a plain (EPI_NONE, bf16) GEMM whose units run first
  // (the long weight-gradient tiles), problem 0 the one with the EPI epilogue; one persistent grid
  // walks both unit lists, so neither problem's wave tail or epilogue is exposed on its own.
  const int U1 = NPROB == 2 ? gs[1].num_units : 0;
  const int total_units = gs[0].num_units + U1;
  constexpr int NUM_EPI_WARPS = epi_warps(EPI);
  using Cfg = GemmCfg<BN, STAGES, PAIR, NUM_EPI_WARPS>;
  constexpr int BMT = PAIR ? 2 * BM : BM;  // tile rows
  constexpr int BNL = PAIR ? BN / 2 : BN;  // B rows staged by this CTA
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ array (not an integer round trip) keeps the shared
  // address space visible to the compiler: LDS / STS instead of generic LD / ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sStg = sB + STAGES * Cfg::B_BYTES;  // NUM_EPI_WARPS x STG_BYTES (1024-aligned)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sStg + NUM_EPI_WARPS * STG_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const int unit0 = PAIR ? (blockIdx.x >> 1) : blockIdx.x;
  const int ustep = PAIR ? (gridDim.x >> 1) : gridDim.x;

  if (warp == 0 && lane == 0) {
    for (int q = 0; q < NPROB; ++q) {
      tma_prefetch_desc(tmA_arr + q);
      tma_prefetch_desc(tmB_arr + q);
    }
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], PAIR ? 2 * NUM_EPI_WARPS : NUM_EPI_WARPS);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
    else tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all();  // peer barriers initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // (the dependents are triggered by the producer once its last loads are issued)
  unsigned long long* trc = (gs[0].trace && blockIdx.x < 2048) ? gs[0].trace + blockIdx.x * 40 : nullptr;
  if (trc && threadIdx.x == 0) trc[0] = gtime_g();
  int tk = 0;  // per-CTA unit counter (trace)

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs of a pair) ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int uu = unit0; uu < total_units; uu += ustep) {
        const int p = (NPROB == 2 && uu < U1) ? 1 : 0;
        const int u = p ? uu : uu - U1;
        const GemmArgs& g = gs[p];
        const CUtensorMap* tmA = tmA_arr + p;
        const CUtensorMap* tmB = tmB_arr + p;
        int tile, kb0, kb1, b1, b2, tm, tn;
        decode_unit(g, u, tile, kb0, kb1);
        decode_tile(g, tile, b1, b2, tm, tn);
        const int arow = tm * BMT + (int)rank * BM;
        const int brow = tn * BN + (int)rank * BNL;
        const int ab1 = g.a_bc1 ? 0 : b1, ab2 = g.a_bc2 ? 0 : b2;
        const int bb1 = g.b_bc1 ? 0 : b1, bb2 = g.b_bc2 ? 0 : b2;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* a_dst = sA + stage * Cfg::A_BYTES;
          uint8_t* b_dst = sB + stage * Cfg::B_BYTES;
          if constexpr (PAIR) {
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::STAGE_BYTES);
            if (!g.a_mn) {
              tma_load_4d_pair(a_dst, tmA, &full_bar[stage], kb * BK, arow, ab1, ab2);
            } else {
#pragma unroll
              for (int i = 0; i < BM / 64; ++i)
                tma_load_4d_pair(a_dst + i * (BK * 128), tmA, &full_bar[stage], arow + i * 64, kb * BK, ab1, ab2);
            }
            if (!g.b_mn) {
              tma_load_4d_pair(b_dst, tmB, &full_bar[stage], kb * BK, brow, bb1, bb2);
            } else {
#pragma unroll
              for (int i = 0; i < BNL / 64; ++i)
                tma_load_4d_pair(b_dst + i * (BK * 128), tmB, &full_bar[stage], brow + i * 64, kb * BK, bb1, bb2);
            }
          } else {
            mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
            if (!g.a_mn) {
              tma_load_4d(a_dst, tmA, &full_bar[stage], kb * BK, arow, ab1, ab2);
            } else {
#pragma unroll
              for (int i = 0; i < BM / 64; ++i)
                tma_load_4d(a_dst + i * (BK * 128), tmA, &full_bar[stage], arow + i * 64, kb * BK, ab1, ab2);
            }
            if (!g.b_mn) {
              tma_load_4d(b_dst, tmB, &full_bar[stage], kb * BK, brow, bb1, bb2);
            } else {
#pragma unroll
              for (int i = 0; i < BNL / 64; ++i)
                tma_load_4d(b_dst + i * (BK * 128), tmB, &full_bar[stage], brow + i * 64, kb * BK, bb1, bb2);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // all operand loads of this CTA issued: what is left is its last MMAs and epilogue, the
      // window in which the next kernel's CTAs may be scheduled (programmatic dependent launch)
      pdl_trigger();
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (the leader CTA of a pair) ----------------
      // The whole warp runs the loop so the descriptor arithmetic stays warp-uniform (uniform
      // registers, no per-MMA R2UR shuffles); one elected lane issues.  Descriptors are built
      // once and advanced by constant offsets (addresses are encoded >> 4 in the low 14 bits).
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int uu = unit0; uu < total_units; uu += ustep) {
        const int p = (NPROB == 2 && uu < U1) ? 1 : 0;
        const int u = p ? uu : uu - U1;
        const GemmArgs& g = gs[p];
        const uint32_t idesc = make_idesc_bf16(BMT, BN, g.a_mn, g.b_mn);
        const uint64_t a_desc0 = make_sw128_desc(smem_u32(sA), g.a_mn ? BK * 128 : 16, 1024);
        const uint64_t b_desc0 = make_sw128_desc(smem_u32(sB), g.b_mn ? BK * 128 : 16, 1024);
        const uint32_t a_kstep = g.a_mn ? (2048 >> 4) : (32 >> 4);
        const uint32_t b_kstep = g.b_mn ? (2048 >> 4) : (32 >> 4);
        int tile, kb0, kb1;
        decode_unit(g, u, tile, kb0, kb1);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        if (trc && lane == 0 && tk < 8) trc[1 + 4 * tk] = gtime_g();
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t a_st = a_desc0 + (uint64_t)((stage * Cfg::A_BYTES) >> 4);
          const uint64_t b_st = b_desc0 + (uint64_t)((stage * Cfg::B_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t adesc = a_st + (uint64_t)(k * a_kstep);
              const uint64_t bdesc = b_st + (uint64_t)(k * b_kstep);
              if constexpr (PAIR) umma_bf16_pair(d_tmem, adesc, bdesc, idesc, (kb != kb0) || (k != 0));
              else umma_bf16(d_tmem, adesc, bdesc, idesc, (kb != kb0) || (k != 0));
            }
            if constexpr (PAIR) umma_commit_pair(&empty_bar[stage], 0x3);
            else umma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) {
          if constexpr (PAIR) umma_commit_pair(&tfull_bar[acc], 0x3);
          else umma_commit(&tfull_bar[acc]);
        }
        __syncwarp();
        if (trc && lane == 0 && tk < 8) trc[2 + 4 * tk] = gtime_g();
        ++tk;
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    // 16 warps: warp % 4 selects the TMEM lane quarter (hardware rule: rows 32*(warp%4)..),
    // (warp - 4) / 4 the column group; a warp owns the 32-column chunks cg, cg+4, ...
    const int quarter = warp & 3;
    const int cgroup = (warp - 4) >> 2;
    constexpr int NGR = NUM_EPI_WARPS / 4;                 // column groups
    constexpr int NCH = BN / 32;                           // 32-column chunks per tile
    constexpr int CPW = NCH >= NGR ? NCH / NGR : 1;        // chunks per warp
    const bool active = cgroup < NCH;                      // small BN: surplus column groups idle
    uint8_t* stg = sStg + (warp - 4) * STG_BYTES;
    int acc = 0;
    uint32_t acc_phase = 0;
    const int etid = threadIdx.x - 128;  // 0 .. 32*NUM_EPI_WARPS-1
    for (int uu = unit0; uu < total_units; uu += ustep) {
      const int p = (NPROB == 2 && uu < U1) ? 1 : 0;
      const int u = p ? uu : uu - U1;
      const GemmArgs& g = gs[p];
      const EpiMaps* maps = maps_arr + p;
      int tile, kb0, kb1, b1, b2, tm, tn;
      decode_unit(g, u, tile, kb0, kb1);
      decode_tile(g, tile, b1, b2, tm, tn);
      const int rl = quarter * 32 + lane;  // row inside this CTA's 128 rows
      const int row0 = tm * BMT + (int)rank * BM + quarter * 32;  // first row of this warp's 32
      const int row = row0 + lane;
      const int64_t c_off = (int64_t)b1 * g.c_bs1 + (int64_t)b2 * g.c_bs2;
      // one tile's epilogue with epilogue kind E (problem 1 of a grouped launch: plain)
      auto tile_epi = [&](auto epi_c) {
        constexpr int E = decltype(epi_c)::value;
        constexpr int EA = E == EPI ? ACT : 0;
        constexpr bool AUXPF = (E == SMPK_EPI_ADD);  // DACT (16 warps, 96 registers) spilled with it
        // DACT / ADD: the auxiliary operand (pre-activation / residual) of the next 32-column chunk
        // is loaded one chunk ahead -- the first one while the main loop still runs -- so its HBM
        // latency is off the epilogue's critical path (ncu r02: 11% of the DACT stall samples)
        uint4 auxv[4];
        auto aux_ok = [&](int i) {
          const int colc = tn * BN + (cgroup + NGR * i) * 32;
          return AUXPF && active && g.splits == 1 && row < g.M && colc + 32 <= g.N && g.vec_ok;
        };
        auto aux_load = [&](int i) {
          if (aux_ok(i)) {
            const uint4* src = reinterpret_cast<const uint4*>(g.aux + c_off + (int64_t)row * g.ldaux + tn * BN +
                                                              (cgroup + NGR * i) * 32);
  #pragma unroll
            for (int q = 0; q < 4; ++q) auxv[q] = __ldg(src + q);
          }
        };
        if constexpr (AUXPF) aux_load(0);

        mbar_wait(&tfull_bar[acc], acc_phase);
        if (trc && warp == 4 && lane == 0 && tk < 8) trc[3 + 4 * tk] = gtime_g();
        tc_fence_after();
        const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16);
        if (g.splits == 1) {
  #pragma unroll 1
          for (int i = 0; i < CPW; ++i) {
            const int ch = cgroup + NGR * i;
            uint32_t r[32];
            if (active) {
              tmem_ld_32x32b_x32(t_row + ch * 32, r);
              tmem_ld_wait();
            }
            if (i == CPW - 1) {  // this warp's accumulator columns are in registers: free the TMEM buffer
              tc_fence_before();
              __syncwarp();
              if (lane == 0) {
                if constexpr (PAIR) mbar_arrive_cluster_relaxed(&tempty_bar[acc], 0);
                else mbar_arrive_relaxed(&tempty_bar[acc]);
              }
            }
            if (!active) continue;
            const int col0 = tn * BN + ch * 32;
            if (col0 >= g.N) continue;
            float v[32];
            uint32_t pre[16];
  #pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            if constexpr (AUXPF) {
              uint4 cur[4];
              const bool have = aux_ok(i);
  #pragma unroll
              for (int q = 0; q < 4; ++q) cur[q] = auxv[q];
              if (i + 1 < CPW) aux_load(i + 1);  // next chunk's operand in flight during this one's math
              epilogue_math32<E, EA, F32OUT, BETA>(g, row < g.M, row, col0, c_off, v, pre, have ? cur : nullptr);
            } else {
              epilogue_math32<E, EA, F32OUT, BETA>(g, row < g.M, row, col0, c_off, v, pre);
            }
            if (g.tma_store) {
              if (lane == 0) bulk_wait_read0();  // the previous chunk's bulk store has read the box
              __syncwarp();
              if constexpr (F32OUT) {
                stage_f32_row(stg, lane, v);
              } else {
                uint32_t w[16];
  #pragma unroll
                for (int j = 0; j < 16; ++j) w[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
                stage_bf16_row(stg, lane, w);
                if constexpr (E == SMPK_EPI_BIAS_ACT) stage_bf16_row(stg + 2048, lane, pre);
              }
              fence_proxy_async_smem();
              __syncwarp();
              if constexpr (!F32OUT) {
                if (g.colsum_part != nullptr && row0 < g.M && col0 + lane < g.N) {  // rows >= M hold zeros
                  // lane = column: sum the box's 32 stored rows (SWIZZLE_64B granule order)
                  float cs4[4] = {0.f, 0.f, 0.f, 0.f};  // 4 independent chains (row order fixed)
  #pragma unroll
                  for (int rr = 0; rr < 32; ++rr) {
                    const bf16* e = reinterpret_cast<const bf16*>(
                        stg + rr * 64 + ((((lane >> 3) ^ ((rr >> 1) & 3))) << 4) + (lane & 7) * 2);
                    cs4[rr & 3] += bf2f(*e);
                  }
                  g.colsum_part[(int64_t)(row0 >> 5) * g.N + col0 + lane] = (cs4[0] + cs4[1]) + (cs4[2] + cs4[3]);
                }
              }
              if (lane == 0) {
                if (g.npeers) {  // reduce-scatter: rows of one CTA belong to one owner
                  const int owner = (int)(row0 / g.rows_per_owner);
                  tma_store_4d(&maps->peer[owner], stg, col0, (int)(row0 - owner * g.rows_per_owner), 0, 0);
                } else {
                  tma_store_4d(&maps->c, stg, col0, row0, b1, b2);
                  if constexpr (E == SMPK_EPI_BIAS_ACT) tma_store_4d(&maps->aux, stg + 2048, col0, row0, b1, b2);
                }
                bulk_commit();
              }
            } else if (row < g.M) {
              epilogue_direct32<E, F32OUT>(g, row, col0, c_off, v, pre);
            }
          }
        } else {
          // split-K: raw fp32 partial of this CTA's 128 x BN block -> ws, column-major inside the
          // block so that a warp's store of one accumulator column is one contiguous 128-byte line
          constexpr int HALVES = PAIR ? 2 : 1;
          const int split = u / g.num_tiles;
          const int sidx = tile * HALVES + (int)rank;  // this CTA's block of the tile
          const int64_t blk = (int64_t)BM * BN;
          float* part = g.ws + ((int64_t)split * g.num_tiles * HALVES + sidx) * blk + rl;
  #pragma unroll 1
          for (int i = 0; i < CPW; ++i) {
            const int ch = cgroup + NGR * i;
            uint32_t r[32];
            if (active) {
              tmem_ld_32x32b_x32(t_row + ch * 32, r);
              tmem_ld_wait();
              float* d = part + (int64_t)ch * 32 * BM;
  #pragma unroll
              for (int j = 0; j < 32; ++j) __stcg(d + j * BM, __uint_as_float(r[j]));
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (PAIR) mbar_arrive_cluster(&tempty_bar[acc], 0);
            else mbar_arrive(&tempty_bar[acc]);
          }
          // all splits of a tile are co-resident (host guarantees num_units <= grid slots): wait
          // for every partial, then this split reduces its stripe of the block's rows in split
          // order (deterministic) and runs the epilogue on it.
          __threadfence();
          named_barrier_sync(1, 32 * NUM_EPI_WARPS);
          if (etid == 0) {
            const int nblk = g.num_tiles * HALVES;
            atomicAdd(g.sem + sidx, 1);
            while (ld_acquire_gpu(g.sem + sidx) < g.splits) __nanosleep(32);
            // last one out re-arms both counters for the next launch
            if (atomicAdd(g.sem + nblk + sidx, 1) == g.splits - 1) {
              g.sem[sidx] = 0;
              g.sem[nblk + sidx] = 0;
            }
          }
          named_barrier_sync(1, 32 * NUM_EPI_WARPS);
          __threadfence();
          const int rows_per = (BM + g.splits - 1) / g.splits;
          const int r0 = split * rows_per;
          const int nrows = min(rows_per, BM - r0);
          const int ngroups = (nrows + 31) >> 5;  // 32-row groups: lane = row
          const int64_t sstride = (int64_t)g.num_tiles * HALVES * blk;
          const float* tbase = g.ws + (int64_t)sidx * blk;
          const int ewarp = etid >> 5;
          for (int item = ewarp; item < ngroups * NCH; item += NUM_EPI_WARPS) {
            const int rg = item / NCH;
            const int ch = item - rg * NCH;
            const int rr = r0 + rg * 32 + lane;
            const int grow = tm * BMT + (int)rank * BM + rr;
            const int col0 = tn * BN + ch * 32;
            if (rr >= r0 + nrows || grow >= g.M || col0 >= g.N) continue;
            float v[32];
  #pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
            const float* src0 = tbase + (int64_t)ch * 32 * BM + rr;
            for (int sp = 0; sp < g.splits; ++sp) {
              const float* src = src0 + sp * sstride;
  #pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += __ldcg(src + j * BM);
            }
            uint32_t pre[16];
            epilogue_math32<E, EA, F32OUT, BETA>(g, true, grow, col0, c_off, v, pre);
            epilogue_direct32<E, F32OUT>(g, grow, col0, c_off, v, pre);
          }
        }
      };
      if (NPROB == 2 && p == 1) tile_epi(std::integral_constant<int, SMPK_EPI_NONE>{});
      else tile_epi(std::integral_constant<int, EPI>{});
      if (trc && warp == 4 && lane == 0 && tk < 8) trc[4 + 4 * tk] = gtime_g();
      ++tk;
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) bulk_wait0();  // bulk stores complete before the CTA (and its smem) retires
  }

  if constexpr (PAIR) {
    tc_fence_before();
    cluster_sync_all();  // both CTAs done with the pair's TMEM and barriers
    if (warp == 2) {
      tc_fence_after();
      tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
    }
  } else {
    __syncthreads();
    if (warp == 2) {
      tc_fence_after();
      tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
  }
}

template <int BN, int STAGES, int EPI, int ACT, bool F32OUT, bool BETA>
__global__ void __launch_bounds__(gemm_threads(EPI), 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ EpiMaps maps, const GemmArgs g) {
  gemm_body<BN, STAGES, EPI, ACT, F32OUT, BETA, false>(&tmA, &tmB, &maps, &g);
}

template <int BN, int STAGES, int EPI, int ACT, bool F32OUT, bool BETA>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gemm_threads(EPI), 1)
    gemm_bf16_tcgen05_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ EpiMaps maps, const GemmArgs g) {
  gemm_body<BN, STAGES, EPI, ACT, F32OUT, BETA, true>(&tmA, &tmB, &maps, &g);
}

// Grouped launch of two independent GEMMs on CTA pairs (see gemm_body NPROB == 2).
struct GroupParams {
  CUtensorMap ta[2], tb[2];
  EpiMaps maps[2];
  GemmArgs g[2];
};

template <int BN, int STAGES, int EPI, int ACT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gemm_threads(EPI), 1)
    gemm_bf16_tcgen05_pair_grouped(const __grid_constant__ GroupParams P) {
  gemm_body<BN, STAGES, EPI, ACT, false, false, true, 2>(P.ta, P.tb, P.maps, P.g);
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
// 4-D tensor map {inner, outer, nb1, nb2} (strides in elements) with boxes {box_inner, box_outer, 1, 1}.
static int make_tma_4d_ex(CUtensorMap* map, const void* ptr, bool f32, CUtensorMapSwizzle swz, int64_t inner,
                          int64_t outer, int64_t ld, int nb1, int64_t s1, int nb2, int64_t s2, int box_inner,
                          int box_outer, const char* name) {
  PFN_encodeTiled_t enc = get_encode_fn();
  const int esz = f32 ? 4 : 2;
  SMPK_REQUIRE(enc != nullptr, SMPK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  SMPK_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, SMPK_ERR_BAD_ARG,
               "operand %s must be 16-byte aligned", name);
  SMPK_REQUIRE((ld * esz) % 16 == 0, SMPK_ERR_BAD_ARG, "leading dim of %s (%lld) must be a multiple of 16 bytes",
               name, (long long)ld);
  SMPK_REQUIRE((nb1 == 1 || (s1 * esz) % 16 == 0) && (nb2 == 1 || (s2 * esz) % 16 == 0), SMPK_ERR_BAD_ARG,
               "batch strides of %s must be multiples of 16 bytes", name);
  cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)nb1, (cuuint64_t)nb2};
  const int64_t fallback = ld * outer * esz;
  cuuint64_t strides[3] = {(cuuint64_t)(ld * esz), (cuuint64_t)(nb1 > 1 ? s1 * esz : fallback),
                           (cuuint64_t)(nb2 > 1 ? s2 * esz : fallback)};
  cuuint32_t box[4] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer, 1u, 1u};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SMPK_REQUIRE(r == CUDA_SUCCESS, SMPK_ERR_CUDA, "tensor map for %s failed (CUresult %d)", name, (int)r);
  return SMPK_OK;
}

// bf16 operand map with SWIZZLE_128B boxes (also used by the attention kernels).
int make_tma_4d(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int nb1, int64_t s1,
                int nb2, int64_t s2, int box_inner, int box_outer, const char* name) {
  return make_tma_4d_ex(map, ptr, false, CU_TENSOR_MAP_SWIZZLE_128B, inner, outer, ld, nb1, s1, nb2, s2, box_inner,
                        box_outer, name);
}

// fp32 map with SWIZZLE_128B boxes (32 fp32 = 128 B inner): the attention backward's ordered dQ
// accumulation (TMA store / reduce-add / load of [box_outer rows x 32 cols] boxes).
int make_tma_4d_f32sw(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                      int box_outer, const char* name) {
  return make_tma_4d_ex(map, ptr, true, CU_TENSOR_MAP_SWIZZLE_128B, inner, outer, ld, 1, 0, 1, 0, box_inner,
                        box_outer, name);
}

// fp32 / 32-bit-word map without swizzle (keep-bit tiles of the attention backward).
int make_tma_4d_b32(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                    int box_outer, const char* name) {
  return make_tma_4d_ex(map, ptr, true, CU_TENSOR_MAP_SWIZZLE_NONE, inner, outer, ld, 1, 0, 1, 0, box_inner,
                        box_outer, name);
}

// TMA-store map of an output [nb2][nb1][rows][cols] with 32 x 32 boxes (see stage_*_row).
static int make_store_map(CUtensorMap* map, const void* ptr, bool f32, int rows, int cols, int64_t ld, int nb1,
                          int64_t s1, int nb2, int64_t s2, const char* name) {
  return make_tma_4d_ex(map, ptr, f32, f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, cols, rows, ld,
                        nb1, s1, nb2, s2, 32, 32, name);
}

// Operand view: rows x K logical, either K-major (K contiguous) or MN-major.
static int make_operand_map(CUtensorMap* map, const void* ptr, bool mn_major, int rows, int K, int64_t ld,
                            int nb1, int64_t s1, int nb2, int64_t s2, int box_rows, const char* name) {
  return make_tma_4d(map, ptr, mn_major ? rows : K, mn_major ? K : rows, ld, nb1, s1, nb2, s2, 64,
                     mn_major ? BK : box_rows, name);
}

// Operand-ring depth: as many stages as fit next to the epilogue staging boxes (max 8).
constexpr int stages_for(int BN, bool pair, int epw) {
  const int stage = BM * BK * 2 + (pair ? BN / 2 : BN) * BK * 2;
  const int budget = 232448 - 1024 - 256 - epw * STG_BYTES;
  return budget / stage < 8 ? budget / stage : 8;
}

template <int BN, int STAGES_UNUSED, bool PAIR, int EPI, int ACT, bool F32OUT, bool BETA>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const EpiMaps& maps, GemmArgs& g,
                       cudaStream_t st) {
  constexpr int STAGES = stages_for(BN, PAIR, epi_warps(EPI));
  using Cfg = GemmCfg<BN, STAGES, PAIR, epi_warps(EPI)>;
  static_assert(Cfg::SMEM_BYTES <= 232448, "shared memory budget");
  auto kern = PAIR ? gemm_bf16_tcgen05_pair<BN, STAGES, EPI, ACT, F32OUT, BETA>
                   : gemm_bf16_tcgen05<BN, STAGES, EPI, ACT, F32OUT, BETA>;
  static unsigned long long attr_set = 0;
  cudaError_t e = smem_attr_once(kern, Cfg::SMEM_BYTES, attr_set);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_gemm: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  const int slots = PAIR ? gemm_sms() / 2 : gemm_sms();  // CTA pairs (one per TPC) or CTAs
  int grid = g.num_units < slots ? g.num_units : slots;
  if (PAIR) grid *= 2;
  launch_pdl(kern, grid, gemm_threads(EPI), Cfg::SMEM_BYTES, st, ta, tb, maps, g);
  return check_launch("smpk_gemm");
}

template <int BN, int STAGES, bool PAIR>
static int dispatch_epilogue(const CUtensorMap& ta, const CUtensorMap& tb, const EpiMaps& maps, GemmArgs& g,
                             cudaStream_t st) {
  const bool beta = g.beta != 0.f;
  switch (g.epi) {
    case SMPK_EPI_NONE:
      if (g.c_f32) return beta ? launch_gemm<BN, STAGES, PAIR, SMPK_EPI_NONE, 0, true, true>(ta, tb, maps, g, st)
                               : launch_gemm<BN, STAGES, PAIR, SMPK_EPI_NONE, 0, true, false>(ta, tb, maps, g, st);
      return beta ? launch_gemm<BN, STAGES, PAIR, SMPK_EPI_NONE, 0, false, true>(ta, tb, maps, g, st)
                  : launch_gemm<BN, STAGES, PAIR, SMPK_EPI_NONE, 0, false, false>(ta, tb, maps, g, st);
    case SMPK_EPI_BIAS:
      if (g.c_f32 || beta) break;
      return launch_gemm<BN, STAGES, PAIR, SMPK_EPI_BIAS, 0, false, false>(ta, tb, maps, g, st);
    case SMPK_EPI_BIAS_ACT:
      if (g.c_f32 || beta) break;
      if (g.act == SMPK_ACT_GELU_ERF) return launch_gemm<BN, STAGES, PAIR, SMPK_EPI_BIAS_ACT, SMPK_ACT_GELU_ERF, false, false>(ta, tb, maps, g, st);
      if (g.act == SMPK_ACT_GELU_TANH) return launch_gemm<BN, STAGES, PAIR, SMPK_EPI_BIAS_ACT, SMPK_ACT_GELU_TANH, false, false>(ta, tb, maps, g, st);
      if (g.act == SMPK_ACT_RELU) return launch_gemm<BN, STAGES, PAIR, SMPK_EPI_BIAS_ACT, SMPK_ACT_RELU, false, false>(ta, tb, maps, g, st);
      break;
    case SMPK_EPI_DACT:
      if (g.c_f32 || beta) break;
      if (g.act == SMPK_ACT_GELU_ERF) return launch_gemm<BN, STAGES, PAIR, SMPK_EPI_DACT, SMPK_ACT_GELU_ERF, false, false>(ta, tb, maps, g, st);
      if (g.act == SMPK_ACT_GELU_TANH) return launch_gemm<BN, STAGES, PAIR, SMPK_EPI_DACT, SMPK_ACT_GELU_TANH, false, false>(ta, tb, maps, g, st);
      if (g.act == SMPK_ACT_RELU) return launch_gemm<BN, STAGES, PAIR, SMPK_EPI_DACT, SMPK_ACT_RELU, false, false>(ta, tb, maps, g, st);
      break;
    case SMPK_EPI_ADD:
      if (g.c_f32 || beta) break;
      return launch_gemm<BN, STAGES, PAIR, SMPK_EPI_ADD, 0, false, false>(ta, tb, maps, g, st);
  }
  set_last_error("smpk_gemm: unsupported epilogue combination epi=%d act=%d c_f32=%d beta=%g", g.epi, g.act, g.c_f32,
                 g.beta);
  return SMPK_ERR_UNSUPPORTED;
}

// Split-K choice (cost model in microseconds): a tile's k-blocks cost t_kb each on one SM;
// splitting adds a fixed sync/fix-up cost and the fp32 partial round trip through L2.
// Splits are only used while every unit fits in one wave (the fix-up waits for all splits
// of a tile, so all of them must be co-resident).
static int choose_splits(int num_tiles, int num_kb, int BN, int nsm, int halves) {
  const double t_kb = 2.0 * BM * BN * BK / 9.0e6;  // us per k-block (~1.33 PFLOP/s over 148 SMs)
  const double t_unit = 1.5, t_fix = 3.0, l2_bytes_per_us = 12.0e6;
  double best = ((num_tiles + nsm - 1) / nsm) * (num_kb * t_kb + t_unit);
  int best_s = 1;
  for (int s = 2; s <= 32 && num_tiles * s <= nsm; ++s) {
    const int kb_per = (num_kb + s - 1) / s;
    if (kb_per < 4) break;
    const int se = (num_kb + kb_per - 1) / kb_per;
    const double t =
        kb_per * t_kb + t_unit + t_fix + 2.0 * se * num_tiles * halves * BM * BN * 4.0 / l2_bytes_per_us;
    if (t < best * 0.95) {
      best = t;
      best_s = se;
    }
  }
  return best_s;
}

// SMPK_GEMM_PAIR=0 disables the CTA-pair kernels (A/B measurements)
static bool pair_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMPK_GEMM_PAIR");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// SMPK_GEMM_PAIR_SPLITK=1 keeps split-K GEMMs on CTA pairs (A/B measurements)
static bool pair_splitk() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMPK_GEMM_PAIR_SPLITK");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

static int pick_bn(int N) { return N <= 64 ? 64 : (N <= 128 ? 128 : 256); }

// Tile plan: CTA pairs (256-row tiles, cta_group::2) whenever N >= 128 and M >= 256, else
// single CTAs; then the split-K count for that tile grid (pairs occupy two SMs per unit).
static void plan_gemm(int M, int N, int K, int nb1, int nb2, int& BN, bool& pair, int& tiles, int& num_kb,
                      int& splits, int& kb_per) {
  BN = pick_bn(N);
  pair = BN >= 128 && M >= 2 * BM && pair_enabled();
  const int rows = pair ? 2 * BM : BM;
  tiles = ((M + rows - 1) / rows) * ((N + BN - 1) / BN) * nb1 * nb2;
  num_kb = (K + BK - 1) / BK;
  splits = choose_splits(tiles, num_kb, BN, pair ? gemm_sms() / 2 : gemm_sms(), pair ? 2 : 1);
  if (pair && splits > 1 && !pair_splitk()) {
    // measured: split-K runs faster on single-CTA tiles (finer units, shorter fix-up)
    pair = false;
    tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN) * nb1 * nb2;
    splits = choose_splits(tiles, num_kb, BN, gemm_sms(), 1);
  }
  kb_per = (num_kb + splits - 1) / splits;
}

// fp32 partial tiles of every (split, tile, CTA of the pair)
static int64_t splitk_ws_bytes(int BN, bool pair, int tiles, int splits) {
  return splits > 1 ? (int64_t)splits * tiles * (pair ? 2 : 1) * BM * BN * 4 : 0;
}

// Per-device split-K arrival counters (zeroed once, re-armed by every launch that uses them);
// each launch takes the next 2*tiles words of a ring so independent GEMMs never share one.
static int* splitk_semaphores(int tiles, int& rc) {
  constexpr int64_t kWords = 1 << 20;
  static int* table[64] = {};
  static int64_t cursor[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  rc = SMPK_OK;
  if (table[dev] == nullptr) {
    void* p = nullptr;
    if (cudaMalloc(&p, kWords * sizeof(int)) != cudaSuccess || cudaMemset(p, 0, kWords * sizeof(int)) != cudaSuccess) {
      set_last_error("smpk_gemm: split-K semaphore table allocation failed (first split-K GEMM inside a graph "
                     "capture? run one eagerly first)");
      rc = SMPK_ERR_CUDA;
      return nullptr;
    }
    table[dev] = reinterpret_cast<int*>(p);
  }
  if (cursor[dev] + 2 * tiles > kWords) cursor[dev] = 0;
  int* s = table[dev] + cursor[dev];
  cursor[dev] += (2 * tiles + 31) & ~31;
  return s;
}

}  // namespace smpk

using namespace smpk;

extern "C" int64_t smpk_gemm_workspace(int M, int N, int K, int nb1, int nb2) {
  if (M <= 0 || N <= 0 || K <= 0 || nb1 <= 0 || nb2 <= 0) return 0;
  int BN, tiles, num_kb, splits, kb_per;
  bool pair;
  plan_gemm(M, N, K, nb1, nb2, BN, pair, tiles, num_kb, splits, kb_per);
  return splitk_ws_bytes(BN, pair, tiles, splits);
}

// Operand / epilogue maps and kernel arguments of one GEMM (no launch).  grouped: the problem runs
// inside a grouped CTA-pair launch, so split-K is off (the other problem fills the machine).
static int gemm_prepare(const void* a, int a_mn_major, int64_t lda, int64_t a_bs1, int64_t a_bs2, const void* b,
                        int b_mn_major, int64_t ldb, int64_t b_bs1, int64_t b_bs2, void* c, int c_f32, int64_t ldc,
                        int64_t c_bs1, int64_t c_bs2, int M, int N, int K, int nb1, int nb2, float alpha, float beta,
                        int epilogue, int act, const void* bias, void* aux, int64_t ldaux, void* const* peers_host,
                        int npeers, int64_t rows_per_owner, int64_t peer_slot_off, void* workspace,
                        int64_t workspace_bytes, float* colsum_part, int grouped, CUtensorMap& ta, CUtensorMap& tb,
                        EpiMaps& maps, GemmArgs& g, int& BN, bool& pair) {
  SMPK_REQUIRE(M > 0 && N > 0 && K > 0 && nb1 > 0 && nb2 > 0, SMPK_ERR_BAD_SHAPE,
               "smpk_gemm: bad shape M=%d N=%d K=%d nb=%dx%d", M, N, K, nb1, nb2);
  SMPK_REQUIRE(a && b && (c || npeers), SMPK_ERR_BAD_ARG, "smpk_gemm: null operand");
  SMPK_REQUIRE(epilogue >= SMPK_EPI_NONE && epilogue <= SMPK_EPI_ADD, SMPK_ERR_BAD_ARG,
               "smpk_gemm: unknown epilogue %d", epilogue);
  const bool need_bias = epilogue == SMPK_EPI_BIAS || epilogue == SMPK_EPI_BIAS_ACT;
  const bool need_aux = epilogue == SMPK_EPI_BIAS_ACT || epilogue == SMPK_EPI_DACT || epilogue == SMPK_EPI_ADD;
  SMPK_REQUIRE(!need_bias || bias, SMPK_ERR_BAD_ARG, "smpk_gemm: epilogue %d needs bias", epilogue);
  SMPK_REQUIRE(!need_aux || aux, SMPK_ERR_BAD_ARG, "smpk_gemm: epilogue %d needs aux", epilogue);
  SMPK_REQUIRE(!(need_aux && c_f32), SMPK_ERR_UNSUPPORTED, "smpk_gemm: aux epilogues need bf16 C");

  int tiles, num_kb, splits, kb_per;
  plan_gemm(M, N, K, nb1, nb2, BN, pair, tiles, num_kb, splits, kb_per);
  if (grouped && splits > 1) {  // back to the CTA-pair plan
    BN = pick_bn(N);
    pair = BN >= 128 && M >= 2 * BM && pair_enabled();
    tiles = ((M + (pair ? 2 * BM : BM) - 1) / (pair ? 2 * BM : BM)) * ((N + BN - 1) / BN) * nb1 * nb2;
    splits = 1;
    kb_per = num_kb;
    if (grouped == 2 && pair) {
      // the grouped launch's plain problem runs its units first: split its long K so that every
      // unit of it still fits in the first wave of CTA pairs (the fix-up needs all splits resident)
      int sp = (gemm_sms() / 2) / tiles;
      while (sp > 1 && (num_kb + sp - 1) / sp < 8) --sp;
      if (sp > 1) {
        kb_per = (num_kb + sp - 1) / sp;
        splits = (num_kb + kb_per - 1) / kb_per;
      }
    }
  }
  if (npeers || splits > 1 && (workspace == nullptr || workspace_bytes < splitk_ws_bytes(BN, pair, tiles, splits))) {
    splits = 1;  // no (or too small a) workspace: single pass over K
    kb_per = num_kb;
  }

  // an operand with batch stride 0 is broadcast over that batch dim (one map slice, coordinate 0)
  const bool a_bc1 = nb1 > 1 && a_bs1 == 0, a_bc2 = nb2 > 1 && a_bs2 == 0;
  const bool b_bc1 = nb1 > 1 && b_bs1 == 0, b_bc2 = nb2 > 1 && b_bs2 == 0;
  int rc = make_operand_map(&ta, a, a_mn_major, M, K, lda, a_bc1 ? 1 : nb1, a_bs1, a_bc2 ? 1 : nb2, a_bs2, BM, "A");
  if (rc) return rc;
  rc = make_operand_map(&tb, b, b_mn_major, N, K, ldb, b_bc1 ? 1 : nb1, b_bs1, b_bc2 ? 1 : nb2, b_bs2,
                        pair ? BN / 2 : BN, "B");
  if (rc) return rc;

  memset(&g, 0, sizeof(g));
  g.M = M;
  g.N = N;
  g.K = K;
  g.nb1 = nb1;
  g.nb2 = nb2;
  g.tiles_m = pair ? (M + 2 * BM - 1) / (2 * BM) : (M + BM - 1) / BM;
  g.tiles_n = (N + BN - 1) / BN;
  g.num_tiles = tiles;
  g.num_kb = num_kb;
  g.splits = splits;
  g.kb_per = kb_per;
  g.num_units = tiles * splits;
  g.ws = reinterpret_cast<float*>(workspace);
  g.sem = nullptr;
  if (splits > 1) {
    SMPK_REQUIRE((reinterpret_cast<uintptr_t>(workspace) & 15) == 0, SMPK_ERR_BAD_ARG,
                 "smpk_gemm: workspace must be 16-byte aligned");
    int rc2;
    g.sem = splitk_semaphores(tiles * (pair ? 2 : 1), rc2);
    if (rc2) return rc2;
  }
  g.a_mn = a_mn_major ? 1 : 0;
  g.a_bc1 = a_bc1;
  g.a_bc2 = a_bc2;
  g.b_bc1 = b_bc1;
  g.b_bc2 = b_bc2;
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
  g.npeers = npeers;
  g.rows_per_owner = rows_per_owner > 0 ? rows_per_owner : 1;
  const int esz = c_f32 ? 4 : 2;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  bool vec = al16(c) && ((ldc * esz) % 16 == 0) && ((c_bs1 * esz) % 16 == 0) && ((c_bs2 * esz) % 16 == 0);
  if (need_bias) vec = vec && al16(bias);
  if (need_aux) vec = vec && al16(aux) && (ldaux % 8 == 0);
  g.vec_ok = vec ? 1 : 0;

  // TMA-store epilogue whenever the outputs are 16-B aligned rows (always for peer stores)
  memset(&maps, 0, sizeof(maps));
  bool tma = false;
  if (npeers) {
    SMPK_REQUIRE(npeers <= MAX_PEERS, SMPK_ERR_BAD_ARG, "smpk_gemm_rs: at most %d peers", MAX_PEERS);
    for (int j = 0; j < npeers; ++j) {
      const bf16* base = reinterpret_cast<const bf16*>(peers_host[j]) + peer_slot_off;
      rc = make_store_map(&maps.peer[j], base, false, (int)rows_per_owner, N, ldc, 1, 0, 1, 0, "peer slot");
      if (rc) return rc;
    }
    tma = true;
  } else if (vec) {
    tma = make_store_map(&maps.c, c, c_f32, M, N, ldc, nb1, c_bs1, nb2, c_bs2, "C") == SMPK_OK;
    if (tma && epilogue == SMPK_EPI_BIAS_ACT)
      tma = make_store_map(&maps.aux, aux, false, M, N, ldaux, nb1, c_bs1, nb2, c_bs2, "aux") == SMPK_OK;
  }
  g.tma_store = tma ? 1 : 0;
  g.colsum_part = colsum_part;
  {
    static int tr = -1;
    static unsigned long long* tp = nullptr;
    if (tr < 0) {
      const char* e = getenv("SMPK_GEMM_TRACE");
      tr = (e && e[0] == '1') ? 1 : 0;
      if (tr) cudaGetSymbolAddress(reinterpret_cast<void**>(&tp), g_gemm_trace);
    }
    g.trace = tr ? tp : nullptr;
  }
  SMPK_REQUIRE(!colsum_part || (tma && !c_f32 && nb1 == 1 && nb2 == 1 && splits == 1), SMPK_ERR_UNSUPPORTED,
               "smpk_gemm: fused column sums need a bf16, unbatched, unsplit TMA-store output");

  return SMPK_OK;
}

static int gemm_impl(const void* a, int a_mn_major, int64_t lda, int64_t a_bs1, int64_t a_bs2, const void* b,
                     int b_mn_major, int64_t ldb, int64_t b_bs1, int64_t b_bs2, void* c, int c_f32, int64_t ldc,
                     int64_t c_bs1, int64_t c_bs2, int M, int N, int K, int nb1, int nb2, float alpha, float beta,
                     int epilogue, int act, const void* bias, void* aux, int64_t ldaux, void* const* peers_host,
                     int npeers, int64_t rows_per_owner, int64_t peer_slot_off, void* workspace,
                     int64_t workspace_bytes, float* colsum_part, void* stream) {
  CUtensorMap ta, tb;
  EpiMaps maps;
  GemmArgs g;
  int BN;
  bool pair;
  int rc = gemm_prepare(a, a_mn_major, lda, a_bs1, a_bs2, b, b_mn_major, ldb, b_bs1, b_bs2, c, c_f32, ldc, c_bs1,
                        c_bs2, M, N, K, nb1, nb2, alpha, beta, epilogue, act, bias, aux, ldaux, peers_host, npeers,
                        rows_per_owner, peer_slot_off, workspace, workspace_bytes, colsum_part, false, ta, tb, maps,
                        g, BN, pair);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // stage counts: stages_for() (fills the 227 KB of shared memory next to the staging boxes)
  if (BN == 64) return dispatch_epilogue<64, 0, false>(ta, tb, maps, g, st);
  if (BN == 128) return pair ? dispatch_epilogue<128, 0, true>(ta, tb, maps, g, st)
                             : dispatch_epilogue<128, 0, false>(ta, tb, maps, g, st);
  return pair ? dispatch_epilogue<256, 0, true>(ta, tb, maps, g, st)
              : dispatch_epilogue<256, 0, false>(ta, tb, maps, g, st);
}

template <int EPI, int ACT>
static int launch_grouped(GroupParams& P, cudaStream_t st) {
  constexpr int BN = 256;
  constexpr int STAGES = stages_for(BN, true, epi_warps(EPI));
  using Cfg = GemmCfg<BN, STAGES, true, epi_warps(EPI)>;
  static_assert(Cfg::SMEM_BYTES <= 232448, "shared memory budget");
  auto kern = gemm_bf16_tcgen05_pair_grouped<BN, STAGES, EPI, ACT>;
  static unsigned long long attr_set = 0;
  cudaError_t e = smem_attr_once(kern, Cfg::SMEM_BYTES, attr_set);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_gemm_grouped: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  const int slots = gemm_sms() / 2;
  const int units = P.g[0].num_units + P.g[1].num_units;
  const int grid = 2 * (units < slots ? units : slots);
  launch_pdl(kern, grid, gemm_threads(EPI), Cfg::SMEM_BYTES, st, P);
  return check_launch("smpk_gemm_grouped");
}

static int desc_impl(const smpk_gemm_desc& d, void* stream) {
  return gemm_impl(d.a, d.a_mn_major, d.lda, d.a_bs1, d.a_bs2, d.b, d.b_mn_major, d.ldb, d.b_bs1, d.b_bs2, d.c,
                   d.c_f32, d.ldc, d.c_bs1, d.c_bs2, d.M, d.N, d.K, d.nb1, d.nb2, d.alpha, d.beta, d.epilogue, d.act,
                   d.bias, d.aux, d.ldaux, nullptr, 0, 0, 0, d.workspace, d.workspace_bytes, d.colsum_part, stream);
}

// mode 1: a grouped problem kept unsplit; mode 2: the grouped launch's plain problem, which may be
// split over K within the first wave (its workspace comes with the descriptor)
static int desc_prepare(const smpk_gemm_desc& d, CUtensorMap& ta, CUtensorMap& tb, EpiMaps& maps, GemmArgs& g,
                        int& BN, bool& pair, int mode = 1) {
  return gemm_prepare(d.a, d.a_mn_major, d.lda, d.a_bs1, d.a_bs2, d.b, d.b_mn_major, d.ldb, d.b_bs1, d.b_bs2, d.c,
                      d.c_f32, d.ldc, d.c_bs1, d.c_bs2, d.M, d.N, d.K, d.nb1, d.nb2, d.alpha, d.beta, d.epilogue,
                      d.act, d.bias, d.aux, d.ldaux, nullptr, 0, 0, 0, mode == 2 ? d.workspace : nullptr,
                      mode == 2 ? d.workspace_bytes : 0, d.colsum_part, mode, ta, tb, maps, g, BN, pair);
}

// SMPK_GEMM_GROUP=0 disables grouped launches (A/B: the same GEMMs launched one after the other)
static bool group_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMPK_GEMM_GROUP");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

extern "C" int smpk_gemm_grouped(const smpk_gemm_desc* descs, int n, void* stream) {
  SMPK_REQUIRE(descs && n >= 1, SMPK_ERR_BAD_ARG, "smpk_gemm_grouped: no problems");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (n == 2 && group_enabled()) {
    // the plain problem (no epilogue, no fused column sums) becomes problem 1
    int q = -1;
    for (int i = 1; i >= 0; --i)
      if (descs[i].epilogue == SMPK_EPI_NONE && !descs[i].colsum_part) q = i;
    bool ok = q >= 0;
    GroupParams P;
    memset(&P, 0, sizeof(P));
    if (ok) {
      const smpk_gemm_desc* d[2] = {&descs[1 - q], &descs[q]};
      for (int i = 0; i < 2 && ok; ++i) {
        int BN;
        bool pair;
        const bool eligible = !d[i]->c_f32 && d[i]->beta == 0.f && d[i]->alpha == 1.f && d[i]->nb1 == 1 &&
                              d[i]->nb2 == 1;
        ok = eligible &&
             desc_prepare(*d[i], P.ta[i], P.tb[i], P.maps[i], P.g[i], BN, pair, i == 1 ? 2 : 1) == SMPK_OK &&
             BN == 256 && pair && (i == 1 || P.g[i].splits == 1) && P.g[i].tma_store;
      }
    }
    // the plain problem's (long, weight-gradient) units must fill at least half the CTA pairs (a
    // small-output wgrad is split over K to get there), and all of them fit in the first wave
    if (ok && (2 * P.g[1].num_units < gemm_sms() / 2 || (P.g[1].splits > 1 && P.g[1].num_units > gemm_sms() / 2)))
      ok = false;
    if (ok) {
      const GemmArgs& g0 = P.g[0];
      switch (g0.epi) {
        case SMPK_EPI_NONE: return launch_grouped<SMPK_EPI_NONE, 0>(P, st);
        case SMPK_EPI_ADD: return launch_grouped<SMPK_EPI_ADD, 0>(P, st);
        case SMPK_EPI_BIAS: return launch_grouped<SMPK_EPI_BIAS, 0>(P, st);
        case SMPK_EPI_DACT:
          if (g0.act == SMPK_ACT_GELU_ERF) return launch_grouped<SMPK_EPI_DACT, SMPK_ACT_GELU_ERF>(P, st);
          if (g0.act == SMPK_ACT_GELU_TANH) return launch_grouped<SMPK_EPI_DACT, SMPK_ACT_GELU_TANH>(P, st);
          if (g0.act == SMPK_ACT_RELU) return launch_grouped<SMPK_EPI_DACT, SMPK_ACT_RELU>(P, st);
          break;
        default:
          break;
      }
    }
  }
  // not groupable: the problems one after the other
  for (int i = 0; i < n; ++i) {
    const int rc = desc_impl(descs[i], stream);
    if (rc) return rc;
  }
  return SMPK_OK;
}

extern "C" int smpk_gemm(const void* a, int a_mn_major, int64_t lda, int64_t a_bs1, int64_t a_bs2, const void* b,
                         int b_mn_major, int64_t ldb, int64_t b_bs1, int64_t b_bs2, void* c, int c_f32,
                         int64_t ldc, int64_t c_bs1, int64_t c_bs2, int M, int N, int K, int nb1, int nb2,
                         float alpha, float beta, int epilogue, int act, const void* bias, void* aux,
                         int64_t ldaux, void* stream) {
  return gemm_impl(a, a_mn_major, lda, a_bs1, a_bs2, b, b_mn_major, ldb, b_bs1, b_bs2, c, c_f32, ldc, c_bs1, c_bs2,
                   M, N, K, nb1, nb2, alpha, beta, epilogue, act, bias, aux, ldaux, nullptr, 0, 0, 0, nullptr, 0,
                   nullptr, stream);
}

extern "C" int smpk_gemm_ex(const void* a, int a_mn_major, int64_t lda, int64_t a_bs1, int64_t a_bs2, const void* b,
                            int b_mn_major, int64_t ldb, int64_t b_bs1, int64_t b_bs2, void* c, int c_f32,
                            int64_t ldc, int64_t c_bs1, int64_t c_bs2, int M, int N, int K, int nb1, int nb2,
                            float alpha, float beta, int epilogue, int act, const void* bias, void* aux,
                            int64_t ldaux, void* workspace, int64_t workspace_bytes, void* stream) {
  return gemm_impl(a, a_mn_major, lda, a_bs1, a_bs2, b, b_mn_major, ldb, b_bs1, b_bs2, c, c_f32, ldc, c_bs1, c_bs2,
                   M, N, K, nb1, nb2, alpha, beta, epilogue, act, bias, aux, ldaux, nullptr, 0, 0, 0, workspace,
                   workspace_bytes, nullptr, stream);
}

extern "C" int64_t smpk_gemm_colsum_rows(int M) { return (M + 31) / 32; }

extern "C" int smpk_gemm_ex2(const void* a, int a_mn_major, int64_t lda, int64_t a_bs1, int64_t a_bs2, const void* b,
                             int b_mn_major, int64_t ldb, int64_t b_bs1, int64_t b_bs2, void* c, int c_f32,
                             int64_t ldc, int64_t c_bs1, int64_t c_bs2, int M, int N, int K, int nb1, int nb2,
                             float alpha, float beta, int epilogue, int act, const void* bias, void* aux,
                             int64_t ldaux, void* workspace, int64_t workspace_bytes, float* colsum_part,
                             void* stream) {
  return gemm_impl(a, a_mn_major, lda, a_bs1, a_bs2, b, b_mn_major, ldb, b_bs1, b_bs2, c, c_f32, ldc, c_bs1, c_bs2,
                   M, N, K, nb1, nb2, alpha, beta, epilogue, act, bias, aux, ldaux, nullptr, 0, 0, 0, workspace,
                   workspace_bytes, colsum_part, stream);
}

extern "C" int smpk_gemm_rs(const void* a, int a_mn_major, int64_t lda, const void* b, int b_mn_major, int64_t ldb,
                            void* const* peers, int npeers, int64_t ldc, int64_t rows_per_owner,
                            int64_t peer_slot_off, int M, int N, int K, void* stream) {
  SMPK_REQUIRE(peers != nullptr && npeers > 0, SMPK_ERR_BAD_ARG, "smpk_gemm_rs: empty peer list");
  SMPK_REQUIRE(rows_per_owner > 0 && rows_per_owner % 128 == 0 && (int64_t)M == rows_per_owner * npeers,
               SMPK_ERR_NOT_DIVISIBLE,
               "smpk_gemm_rs: M=%d must be %d owners x rows per owner (%lld, a multiple of 128)", M, npeers,
               (long long)rows_per_owner);
  return gemm_impl(a, a_mn_major, lda, 0, 0, b, b_mn_major, ldb, 0, 0, nullptr, 0, ldc, 0, 0, M, N, K, 1, 1, 1.f,
                   0.f, SMPK_EPI_NONE, 0, nullptr, nullptr, 0, peers, npeers, rows_per_owner, peer_slot_off, nullptr,
                   0, nullptr, stream);
}

extern "C" int smpk_debug_gemm_trace(void* host_out, int n_cta) {
  if (n_cta > 2048) n_cta = 2048;
  cudaError_t e = cudaMemcpyFromSymbol(host_out, smpk::g_gemm_trace, (size_t)n_cta * 40 * 8);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_debug_gemm_trace: %s", cudaGetErrorString(e));
  return SMPK_OK;
}

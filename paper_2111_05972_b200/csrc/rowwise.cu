// rowwise.cu — HBM-bound row kernels of the transformer layer (sm_100a).
//
//   smpk_bdr_ln_fwd  : r = residual + dropout(x + bias);  y = LayerNorm(r)   (K7+K8+K9 fused)
//   smpk_ln_bwd      : dr = LN'(dy) + dres;  dsub = dropout'(dr);  dgamma/dbeta/dbias column sums
//   smpk_softmax_fwd : P = softmax(scale*S + mask [+causal]);  Pd = dropout(P)              (K6+K9)
//   smpk_softmax_bwd : dS = scale * (Pd*dPd - P*sum(Pd*dPd))
//   smpk_colsum      : deterministic column sums (bias gradients)
//
// 128-bit vectorised loads/stores, warp-shuffle reductions, row groups of W warps
// (W*256*VPT = H) so each lane keeps its slice of the row in registers.  Every
// reduction runs in a fixed order, so results are bit-stable run to run.
// Dropout masks come from Philox4x32-10 keyed by logical coordinates
// (oracle/philox.py reproduces them bit-exactly).
#include <cstdlib>

#include "smpk_common.cuh"

namespace smpk {

constexpr int ROW_THREADS = 256;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Sum over the W warps of one row group, fixed order (deterministic).
template <int W>
__device__ __forceinline__ float group_sum(float v, float* sm, int slot, int wi) {
  v = warp_sum(v);
  if constexpr (W == 1) {
    return v;
  } else {
    if ((threadIdx.x & 31) == 0) sm[slot * W + wi] = v;
    named_bar(1 + slot, W * 32);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < W; ++i) s += sm[slot * W + i];
    named_bar(1 + slot, W * 32);
    return s;
  }
}

// Two sums over the W warps of one row group at once (one barrier round instead of two).
template <int W>
__device__ __forceinline__ float2 group_sum2(float2 v, float* sm, int slot, int wi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  if constexpr (W == 1) {
    return v;
  } else {
    if ((threadIdx.x & 31) == 0) reinterpret_cast<float2*>(sm)[slot * W + wi] = v;
    named_bar(1 + slot, W * 32);
    float2 s = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const float2 t = reinterpret_cast<const float2*>(sm)[slot * W + i];
      s.x += t.x;
      s.y += t.y;
    }
    named_bar(1 + slot, W * 32);
    return s;
  }
}

// Bulk L2 prefetch of a contiguous 16-byte-aligned span (no registers held; the row kernels use it
// to pull the next row's inputs toward L2 while the current row computes).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  if ((reinterpret_cast<uintptr_t>(p) | bytes) & 15u) return;  // the bulk form needs 16-byte granules
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void unpack8(const uint4 u, float (&v)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = unpack_bf16x2(w[j]);
    v[2 * j] = f.x;
    v[2 * j + 1] = f.y;
  }
}
__device__ __forceinline__ void load8(const bf16* p, float (&v)[8]) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 f = unpack_bf16x2(w[j]);
    v[2 * j] = f.x;
    v[2 * j + 1] = f.y;
  }
}
__device__ __forceinline__ void store8(bf16* p, const float (&v)[8]) {
  uint4 u;
  u.x = pack_bf16x2(v[0], v[1]);
  u.y = pack_bf16x2(v[2], v[3]);
  u.z = pack_bf16x2(v[4], v[5]);
  u.w = pack_bf16x2(v[6], v[7]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void round8_int(float (&v)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = round_bf16(v[j]);
}

// bf16 round-to-nearest-even kept in fp32: one cvt.rn.bf16x2 per pair + unpack (the row
// kernels are not XU-bound, unlike the GEMM epilogue that keeps the integer form)
__device__ __forceinline__ void round8(float (&v)[8]) {
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float2 f = unpack_bf16x2(pack_bf16x2(v[j], v[j + 1]));
    v[j] = f.x;
    v[j + 1] = f.y;
  }
}

// keep flags of 8 columns: from the stored keep byte (bit j = column j) when the forward
// saved it, else from Philox
__device__ __forceinline__ void keep8_from_byte(uint32_t byte, bool (&keep)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) keep[j] = (byte >> j) & 1u;
}
__device__ __forceinline__ uint32_t keep8_to_byte(const bool (&keep)[8]) {
  uint32_t b = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) b |= (keep[j] ? 1u : 0u) << j;
  return b;
}

struct RowGeom {
  int W, VPT;
};

// Prefer <= 2 uint4 chunks per lane (register pressure / occupancy of the
// memory-bound row kernels), spreading a row over up to 8 warps.
// H need only be a multiple of 8: the last 256-column chunk may be partial (lanes past H idle),
// which the channel-sharded (memory-mode) widths H/T and 3H/T need.
static bool row_geom(int H, RowGeom& g) {
  if (H <= 0 || H % 8) return false;
  const int n = (H + 255) / 256;
  for (int W = 1; W <= 8; W *= 2) {
    if (n % W) continue;
    const int v = n / W;
    if (v <= 2) {
      g.W = W;
      g.VPT = v;
      return true;
    }
  }
  for (int W = 1; W <= 8; W *= 2) {
    if (n % W) continue;
    const int v = n / W;
    if (v <= 5 || (W == 8 && v <= 8)) {
      g.W = W;
      g.VPT = v;
      return true;
    }
  }
  return false;
}

static bool fast_enabled() {  // SMPK_ROW_FAST=0: the general row kernels only (A/B)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMPK_ROW_FAST");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v != 0;
}

static int row_grid(int M, int W, int ctas_per_sm = 4) {
  const int rows_per_cta = (ROW_THREADS / 32) / W;
  int need = (M + rows_per_cta - 1) / rows_per_cta;
  int cap = row_sms() * ctas_per_sm;
  return need < cap ? need : cap;
}

// ===========================================================================
// bias + dropout + residual + LayerNorm forward
// ===========================================================================
struct BdrLnArgs {
  const bf16* x;
  const bf16* bias;
  const bf16* residual;
  bf16* r_out;
  const bf16* gamma;
  const bf16* beta;
  bf16* y_out;
  float* mean;
  float* rstd;
  int M, H;
  float eps, p;
  uint64_t seed;
  uint32_t layer, site;
  int64_t row_offset;
  // reduce-scatter consumer: x = sum_{j < nslots} x[j * slot_stride + ...] (ascending rank)
  int nslots;
  int64_t slot_stride;
  // allgather producer: the final output (y, or r without LN) is also stored to every
  // peer-mapped buffer out_peers[j] + peer_off (NVLink peer stores)
  bf16* const* out_peers;
  int npeers;
  int64_t peer_off;
  // channel-sharded LayerNorm (memory mode): dropout column offset of this shard; partial
  // row sums (sum r, sum r^2 over the local columns) out; or the group's row sums in
  int64_t col_offset;
  float* row_sums_out;
  const float* ext_sums;
  int H_total;
  uint8_t* keep_out;  // [M][H/8] hidden-dropout keep bytes for the backward (may be null)
  // x read as the ascending-rank sum over the nslots peers' buffers x_peers[j] + x_peer_off
  const bf16* const* x_peers;
  int64_t x_peer_off;
  const uint64_t* rng_step = nullptr;  // device step word: Philox key = seed + step * golden (may be null)
};

__device__ __forceinline__ void load8_slots(const bf16* p, int nslots, int64_t stride, float (&v)[8]) {
  load8(p, v);
  for (int j = 1; j < nslots; ++j) {
    float t[8];
    load8(p + j * stride, t);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] += t[e];
  }
}

// reduce-scatter consumer over peer memory (pull): the ascending-rank sum of the T ranks'
// partial rows, rank j's at peers[j] + off (its own GEMM output in its symmetric pool)
__device__ __forceinline__ void load8_peer_slots(const bf16* const* peers, int n, int64_t off, float (&v)[8]) {
  // sequential (few registers: these kernels keep per-column accumulators in registers; the
  // bandwidth-critical pull path is the pipelined bulk-copy kernel)
  load8(peers[0] + off, v);
  for (int j = 1; j < n; ++j) {
    float t[8];
    load8(peers[j] + off, t);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] += t[e];
  }
}

__device__ __forceinline__ void store8_peers(bf16* const* peers, int npeers, int64_t off, const float (&v)[8]) {
  uint4 u;
  u.x = pack_bf16x2(v[0], v[1]);
  u.y = pack_bf16x2(v[2], v[3]);
  u.z = pack_bf16x2(v[4], v[5]);
  u.w = pack_bf16x2(v[6], v[7]);
  for (int j = 0; j < npeers; ++j) *reinterpret_cast<uint4*>(peers[j] + off) = u;
}

template <int W, int VPT>
__global__ void __launch_bounds__(ROW_THREADS) bdr_ln_fwd_kernel(const BdrLnArgs a) {
  pdl_trigger();
  pdl_wait();
  const uint64_t pkey = philox_key(a.seed, a.rng_step);
  __shared__ float sm[2 * 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp / W, wi = warp % W;
  const int rows_per_cta = (ROW_THREADS / 32) / W;
  const float inv_keep = a.p > 0.f ? 1.f / (1.f - a.p) : 1.f;
  // Single-slot local input: the next row's x / residual are loaded into registers before this
  // row's dropout / statistics / stores, so a row's math overlaps the next row's HBM latency.
  const bool prefetch = a.x_peers == nullptr && a.nslots == 1;
  const int row_step = gridDim.x * rows_per_cta;
  uint4 px[VPT], pr[VPT];
  auto issue = [&](int row) {
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int col = ((i * W + wi) * 32 + lane) * 8;
      if (row < a.M && col < a.H) {
        px[i] = *reinterpret_cast<const uint4*>(a.x + (int64_t)row * a.H + col);
        if (a.residual) pr[i] = *reinterpret_cast<const uint4*>(a.residual + (int64_t)row * a.H + col);
      }
    }
  };
  if (prefetch) issue(blockIdx.x * rows_per_cta + slot);
  for (int row0 = blockIdx.x * rows_per_cta; row0 < a.M; row0 += row_step) {
    const int row = row0 + slot;
    const bool valid = row < a.M;
    float v[VPT][8], res[VPT][8];
    // every load of the row first (memory-level parallelism), then the math
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int col = ((i * W + wi) * 32 + lane) * 8;
      if (prefetch) {
        if (valid && col < a.H) {
          unpack8(px[i], v[i]);
          if (a.residual) unpack8(pr[i], res[i]);
        }
      } else if (valid && col < a.H) {
        if (a.x_peers)
          load8_peer_slots(a.x_peers, a.nslots, a.x_peer_off + (int64_t)row * a.H + col, v[i]);
        else
          load8_slots(a.x + (int64_t)row * a.H + col, a.nslots, a.slot_stride, v[i]);
        if (a.residual) load8(a.residual + (int64_t)row * a.H + col, res[i]);
      }
    }
    if (prefetch) issue(row + row_step);
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int col = ((i * W + wi) * 32 + lane) * 8;
      if (valid && col < a.H) {
        if (a.bias) {
          float b[8];
          load8(a.bias + col, b);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[i][j] += b[j];
        }
        if (a.p > 0.f) {
          bool keep[8];
          dropout_keep8(pkey, a.layer, a.site, (uint64_t)(a.row_offset + row), (int)(a.col_offset + col),
                        dropout_threshold(a.p), keep);
          if (a.keep_out) a.keep_out[(int64_t)row * (a.H / 8) + col / 8] = (uint8_t)keep8_to_byte(keep);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[i][j] = keep[j] ? v[i][j] * inv_keep : 0.f;
        }
        if (a.residual) {
#pragma unroll
          for (int j = 0; j < 8; ++j) v[i][j] += res[i][j];
        }
        round8(v[i]);
        if (a.r_out) store8(a.r_out + (int64_t)row * a.H + col, v[i]);
        if (a.npeers && a.gamma == nullptr) store8_peers(a.out_peers, a.npeers, a.peer_off + (int64_t)row * a.H + col, v[i]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[i][j] = 0.f;
      }
    }
    if (a.row_sums_out) {  // partial row sums of r over this shard's columns (uniform branch)
      float s = 0.f, q = 0.f;
#pragma unroll
      for (int i = 0; i < VPT; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s += v[i][j];
          q += v[i][j] * v[i][j];
        }
      s = group_sum<W>(s, sm, slot, wi);
      q = group_sum<W>(q, sm + 8, slot, wi);
      if (valid && wi == 0 && lane == 0) {
        a.row_sums_out[2 * (int64_t)row] = s;
        a.row_sums_out[2 * (int64_t)row + 1] = q;
      }
    }
    if (a.gamma == nullptr) continue;  // uniform across the CTA
    float mu, var;
    if (a.ext_sums) {  // the TP group's row sums: mean = S1/n, var = S2/n - mean^2
      mu = valid ? a.ext_sums[2 * (int64_t)row] / a.H_total : 0.f;
      var = valid ? fmaxf(a.ext_sums[2 * (int64_t)row + 1] / a.H_total - mu * mu, 0.f) : 0.f;
    } else {
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < VPT; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += v[i][j];
      mu = group_sum<W>(s, sm, slot, wi) / a.H;
      float q = 0.f;
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        if (((i * W + wi) * 32 + lane) * 8 >= a.H) continue;  // idle lanes of a partial chunk
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float d = v[i][j] - mu;
          q += d * d;
        }
      }
      var = group_sum<W>(q, sm + 8, slot, wi) / a.H;
    }
    const float rs = rsqrtf(var + a.eps);
    if (valid) {
      if (wi == 0 && lane == 0) {
        a.mean[row] = mu;
        a.rstd[row] = rs;
      }
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int col = ((i * W + wi) * 32 + lane) * 8;
        if (col >= a.H) continue;
        float gm[8], bt[8], o[8];
        load8(a.gamma + col, gm);
        load8(a.beta + col, bt);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = (v[i][j] - mu) * rs * gm[j] + bt[j];
        if (a.y_out) store8(a.y_out + (int64_t)row * a.H + col, o);
        if (a.npeers) store8_peers(a.out_peers, a.npeers, a.peer_off + (int64_t)row * a.H + col, o);
      }
    }
  }
}

// Local fast path of bdr_ln_fwd (one input slot, no peers, bias + residual + LayerNorm, whole
// 256-column chunks): the flags the general kernel tests per chunk are fixed, bias / gamma / beta
// are re-read per row from L1 (holding them in registers spilled at 3 CTAs per SM), and the fp32
// math runs as paired FFMA2 / FADD2 / FMUL2.  The general kernel issued ~58 instructions per
// element here (ncu: issue-bound at 62 %).
__device__ __forceinline__ float2 bf2f(uint32_t w) { return unpack_bf16x2(w); }

template <int W, int VPT, bool BR, bool LN>
__global__ void __launch_bounds__(ROW_THREADS, 3) bdr_ln_fwd_fast_kernel(const BdrLnArgs a) {
  // BR: bias + dropout + residual (else r = x); LN: LayerNorm statistics and y (else r only)
  pdl_trigger();
  pdl_wait();
  const uint64_t pkey = philox_key(a.seed, a.rng_step);
  const PhiloxRoundKeys rk = philox_round_keys(static_cast<uint32_t>(pkey), static_cast<uint32_t>(pkey >> 32));
  __shared__ float sm[2 * 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp / W, wi = warp % W;
  const int rows_per_cta = (ROW_THREADS / 32) / W;
  const bool drop = BR && a.p > 0.f;
  const float ik = drop ? 1.f / (1.f - a.p) : 1.f;
  const uint32_t thresh = dropout_threshold(a.p);
  const int row_step = gridDim.x * rows_per_cta;
  const float inv_h = 1.f / a.H;
  int col[VPT];
#pragma unroll
  for (int i = 0; i < VPT; ++i) col[i] = ((i * W + wi) * 32 + lane) * 8;
  uint4 px[VPT], pr[VPT];
  auto issue = [&](int row) {
    if (row < a.M) {
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        px[i] = *reinterpret_cast<const uint4*>(a.x + (int64_t)row * a.H + col[i]);
        if (BR) pr[i] = *reinterpret_cast<const uint4*>(a.residual + (int64_t)row * a.H + col[i]);
      }
    }
  };
  issue(blockIdx.x * rows_per_cta + slot);
  const float2 ik2 = make_float2(ik, ik);
  for (int row0 = blockIdx.x * rows_per_cta; row0 < a.M; row0 += row_step) {
    const int row = row0 + slot;
    const bool valid = row < a.M;
    float2 v[VPT][4];
    float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const uint32_t xw[4] = {px[i].x, px[i].y, px[i].z, px[i].w};
      if (!BR) {  // r = x (already bf16)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[i][j] = bf2f(xw[j]);
          s2 = __fadd2_rn(s2, v[i][j]);
        }
        if (valid && a.r_out) *reinterpret_cast<uint4*>(a.r_out + (int64_t)row * a.H + col[i]) = px[i];
        continue;
      }
      const uint32_t rw[4] = {pr[i].x, pr[i].y, pr[i].z, pr[i].w};
      const uint4 bb = *reinterpret_cast<const uint4*>(a.bias + col[i]);  // L1-resident across rows
      const uint32_t bw[4] = {bb.x, bb.y, bb.z, bb.w};
      uint32_t kbyte = 0xffu;
      u32x4 ph = {0u, 0u, 0u, 0u};
      if (drop && valid) {
        const u32x4 c = {static_cast<uint32_t>(col[i] >> 3), static_cast<uint32_t>(a.row_offset + row), a.layer,
                         a.site};
        ph = philox4x32_10(c, rk);
      }
      const uint32_t pw[4] = {ph.x, ph.y, ph.z, ph.w};
      if (drop) kbyte = 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 t = __fadd2_rn(bf2f(xw[j]), bf2f(bw[j]));
        if (drop) {
          const bool k0 = (pw[j] & 0xffffu) >= thresh, k1 = (pw[j] >> 16) >= thresh;
          kbyte |= (k0 ? 1u : 0u) << (2 * j);
          kbyte |= (k1 ? 1u : 0u) << (2 * j + 1);
          t = __fmul2_rn(t, ik2);
          t.x = k0 ? t.x : 0.f;
          t.y = k1 ? t.y : 0.f;
        }
        t = __fadd2_rn(t, bf2f(rw[j]));
        t = bf2f(pack_bf16x2(t.x, t.y));  // r in bf16
        v[i][j] = t;
        s2 = __fadd2_rn(s2, t);
      }
      if (valid && a.keep_out) a.keep_out[(int64_t)row * (a.H / 8) + col[i] / 8] = (uint8_t)kbyte;
      if (valid && a.r_out) {
        uint4 u;
        u.x = pack_bf16x2(v[i][0].x, v[i][0].y);
        u.y = pack_bf16x2(v[i][1].x, v[i][1].y);
        u.z = pack_bf16x2(v[i][2].x, v[i][2].y);
        u.w = pack_bf16x2(v[i][3].x, v[i][3].y);
        *reinterpret_cast<uint4*>(a.r_out + (int64_t)row * a.H + col[i]) = u;
      }
    }
    issue(row + row_step);  // next row's loads overlap this row's statistics and stores
    if (!LN) continue;
    const float mu = group_sum<W>(s2.x + s2.y, sm, slot, wi) * inv_h;
    const float2 nmu = make_float2(-mu, -mu);
    float2 q2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < VPT; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[i][j] = __fadd2_rn(v[i][j], nmu);
        q2 = __ffma2_rn(v[i][j], v[i][j], q2);
      }
    const float var = group_sum<W>(q2.x + q2.y, sm + 8, slot, wi) * inv_h;
    const float rs = rsqrtf(var + a.eps);
    const float2 rs2 = make_float2(rs, rs);
    if (valid) {
      if (wi == 0 && lane == 0) {
        a.mean[row] = mu;
        a.rstd[row] = rs;
      }
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const uint4 gg = *reinterpret_cast<const uint4*>(a.gamma + col[i]);
        const uint4 be = *reinterpret_cast<const uint4*>(a.beta + col[i]);
        const uint32_t gw[4] = {gg.x, gg.y, gg.z, gg.w};
        const uint32_t ew[4] = {be.x, be.y, be.z, be.w};
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 t = __ffma2_rn(__fmul2_rn(v[i][j], rs2), bf2f(gw[j]), bf2f(ew[j]));
          o[j] = pack_bf16x2(t.x, t.y);
        }
        *reinterpret_cast<uint4*>(a.y_out + (int64_t)row * a.H + col[i]) = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
  }
}

// ===========================================================================
// LayerNorm backward (+ residual grad, + dropout backward, + column partials)
// ===========================================================================
struct LnBwdArgs {
  const bf16* dy;
  const bf16* r;
  const float* mean;
  const float* rstd;
  const bf16* gamma;
  const bf16* dres;
  bf16* dr_out;
  bf16* dsub_out;
  float* partials;  // [gridDim.x][3][H]: dgamma, dbeta, dbias
  int M, H;
  float p;
  uint64_t seed;
  uint32_t layer, site;
  int64_t row_offset;
  int nslots;          // dy = sum of nslots partial slots (reduce-scatter consumer)
  int64_t slot_stride;
  bf16* const* out_peers;  // dsub also stored to every peer buffer (allgather producer)
  int npeers;
  int64_t peer_off;
  // channel-sharded LayerNorm (memory mode): dropout column offset; sums-only pass writing the
  // partial row sums (sum g, sum g*xhat; g = dy*gamma) of the local columns; or the group's sums in
  int64_t col_offset;
  float* row_sums_out;
  const float* ext_sums;
  int H_total;
  const uint8_t* keep_in;  // [M][H/8] keep bytes saved by the forward (null: recompute Philox)
  const bf16* const* dy_peers;  // dy = ascending-rank sum over dy_peers[j] + dy_peer_off (pull)
  int64_t dy_peer_off;
  const uint64_t* rng_step = nullptr;
};

template <int W, int VPT>
__device__ __forceinline__ void flush_partial(const float (&acc)[VPT][8], float* out, float* red, int nslots, int slot,
                                              int wi, int lane, int H) {
  if (nslots == 1) {
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      if (((i * W + wi) * 32 + lane) * 8 >= H) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j) out[((i * W + wi) * 32 + lane) * 8 + j] = acc[i][j];
    }
    return;
  }
  float* buf = red + wi * (VPT * 8 * 32);
  for (int sl = 0; sl < nslots; ++sl) {
    if (slot == sl) {
#pragma unroll
      for (int i = 0; i < VPT; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float* d = buf + (i * 8 + j) * 32 + lane;
          *d = (sl == 0) ? acc[i][j] : *d + acc[i][j];
        }
    }
    __syncthreads();
  }
  if (slot == nslots - 1) {
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      if (((i * W + wi) * 32 + lane) * 8 >= H) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j) out[((i * W + wi) * 32 + lane) * 8 + j] = buf[(i * 8 + j) * 32 + lane];
    }
  }
  __syncthreads();
}

template <int W, int VPT>
__global__ void __launch_bounds__(ROW_THREADS) ln_bwd_kernel(const LnBwdArgs a) {
  pdl_trigger();
  pdl_wait();
  const uint64_t pkey = philox_key(a.seed, a.rng_step);
  __shared__ float sm[2 * 8];
  extern __shared__ float red[];  // [W][VPT*8][32] slot reduction buffer
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp / W, wi = warp % W;
  const int rows_per_cta = (ROW_THREADS / 32) / W;
  const float inv_keep = a.p > 0.f ? 1.f / (1.f - a.p) : 1.f;
  const bool has_ln = a.gamma != nullptr;  // no-LN mode: d = dy (+ dres)
  float acc_g[VPT][8], acc_b[VPT][8], acc_d[VPT][8];
#pragma unroll
  for (int i = 0; i < VPT; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc_g[i][j] = acc_b[i][j] = acc_d[i][j] = 0.f;

  for (int row0 = blockIdx.x * rows_per_cta; row0 < a.M; row0 += gridDim.x * rows_per_cta) {
    const int row = row0 + slot;
    const bool valid = row < a.M;
    {  // next row of this slot: dy / r / dres / keep bytes toward L2 (registers are the limiter here)
      const int nrow = row + gridDim.x * rows_per_cta;
      if (wi == 0 && lane == 0 && nrow < a.M) {
        const uint32_t rb = (uint32_t)a.H * 2;
        if (a.dy_peers == nullptr && a.nslots == 1) prefetch_l2(a.dy + (int64_t)nrow * a.H, rb);
        if (has_ln) prefetch_l2(a.r + (int64_t)nrow * a.H, rb);
        if (a.dres) prefetch_l2(a.dres + (int64_t)nrow * a.H, rb);
        if (a.keep_in) prefetch_l2(a.keep_in + (int64_t)nrow * (a.H / 8), a.H / 8);
      }
    }
    float xh[VPT][8], g[VPT][8];
    float mu = 0.f, rs = 0.f;
    if (valid && has_ln) {
      mu = a.mean[row];
      rs = a.rstd[row];
    }
    float s1 = 0.f, s2 = 0.f;
    uint4 dres_raw[VPT];  // residual-gradient loads issued with the others (memory-level parallelism)
    uint32_t keep_raw[VPT];  // stored keep bytes, likewise loaded up front
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int col = ((i * W + wi) * 32 + lane) * 8;
      if (valid && a.dres && col < a.H)
        dres_raw[i] = *reinterpret_cast<const uint4*>(a.dres + (int64_t)row * a.H + col);
      keep_raw[i] = (valid && a.keep_in && col < a.H) ? a.keep_in[(int64_t)row * (a.H / 8) + col / 8] : 0u;
    }
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int col = ((i * W + wi) * 32 + lane) * 8;
      if (valid && col < a.H && !has_ln) {
        if (a.dy_peers)
          load8_peer_slots(a.dy_peers, a.nslots, a.dy_peer_off + (int64_t)row * a.H + col, g[i]);
        else
          load8_slots(a.dy + (int64_t)row * a.H + col, a.nslots, a.slot_stride, g[i]);
      } else if (valid && col < a.H) {
        float dy[8], gm[8];
        load8(a.r + (int64_t)row * a.H + col, xh[i]);
        if (a.dy_peers)
          load8_peer_slots(a.dy_peers, a.nslots, a.dy_peer_off + (int64_t)row * a.H + col, dy);
        else
          load8_slots(a.dy + (int64_t)row * a.H + col, a.nslots, a.slot_stride, dy);
        load8(a.gamma + col, gm);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          xh[i][j] = (xh[i][j] - mu) * rs;
          g[i][j] = dy[j] * gm[j];
          s1 += g[i][j];
          s2 += g[i][j] * xh[i][j];
          acc_g[i][j] += dy[j] * xh[i][j];
          acc_b[i][j] += dy[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) xh[i][j] = g[i][j] = 0.f;
      }
    }
    float m1, m2;
    if (a.ext_sums) {
      m1 = valid ? a.ext_sums[2 * (int64_t)row] / a.H_total : 0.f;
      m2 = valid ? a.ext_sums[2 * (int64_t)row + 1] / a.H_total : 0.f;
    } else {
      m1 = group_sum<W>(s1, sm, slot, wi);
      m2 = group_sum<W>(s2, sm + 8, slot, wi);
      if (a.row_sums_out) {  // sums-only pass (uniform branch)
        if (valid && wi == 0 && lane == 0) {
          a.row_sums_out[2 * (int64_t)row] = m1;
          a.row_sums_out[2 * (int64_t)row + 1] = m2;
        }
        continue;
      }
      m1 /= a.H;
      m2 /= a.H;
    }
    if (!valid) continue;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int col = ((i * W + wi) * 32 + lane) * 8;
      if (col >= a.H) continue;  // idle lanes of a partial chunk
      float d[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) d[j] = has_ln ? rs * (g[i][j] - m1 - xh[i][j] * m2) : g[i][j];
      if (a.dres) {
        const uint32_t w[4] = {dres_raw[i].x, dres_raw[i].y, dres_raw[i].z, dres_raw[i].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = unpack_bf16x2(w[j]);
          d[2 * j] += f.x;
          d[2 * j + 1] += f.y;
        }
      }
      round8(d);
      if (a.dr_out) store8(a.dr_out + (int64_t)row * a.H + col, d);
      if (a.p > 0.f) {
        bool keep[8];
        if (a.keep_in)
          keep8_from_byte(keep_raw[i], keep);
        else
          dropout_keep8(pkey, a.layer, a.site, (uint64_t)(a.row_offset + row), (int)(a.col_offset + col),
                        dropout_threshold(a.p), keep);
#pragma unroll
        for (int j = 0; j < 8; ++j) d[j] = keep[j] ? d[j] * inv_keep : 0.f;
        round8(d);
        store8(a.dsub_out + (int64_t)row * a.H + col, d);
      }
      if (a.npeers) store8_peers(a.out_peers, a.npeers, a.peer_off + (int64_t)row * a.H + col, d);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc_d[i][j] += d[j];
    }
  }
  // CTA partials: warps with the same wi own the same columns; slots are summed
  // in ascending order through shared memory (deterministic).
  if (a.row_sums_out) return;  // sums-only pass: no column partials
  float* out = a.partials + (int64_t)blockIdx.x * 3 * a.H;
  flush_partial<W, VPT>(acc_g, out, red, rows_per_cta, slot, wi, lane, a.H);
  flush_partial<W, VPT>(acc_b, out + a.H, red, rows_per_cta, slot, wi, lane, a.H);
  flush_partial<W, VPT>(acc_d, out + 2 * a.H, red, rows_per_cta, slot, wi, lane, a.H);
}

// Reduce P partial rows of [P][K][H] to K outputs of H columns (fixed order).
// block = 32 columns x NG row groups; each thread sums every NG-th partial row (4 independent
// accumulators), then the NG group sums are added in ascending order (deterministic).  NG = 32
// for long partial lists: ~4x fewer dependent load round trips per thread than NG = 8.
template <int NG>
__global__ void __launch_bounds__(32 * NG) colsum_reduce_kernel(const float* partials, int P, int K, int H, void* o0,
                                                                void* o1, void* o2, int out_f32, int accumulate) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sm[NG][33];
  const int c = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + c;
  const int k = blockIdx.y;
  void* o = k == 0 ? o0 : (k == 1 ? o1 : o2);
  if (o == nullptr) return;  // uniform per block
  float part = 0.f;
  if (col < H) {
    float q[4] = {0.f, 0.f, 0.f, 0.f};
    int p = grp;
    for (; p + 3 * NG < P; p += 4 * NG) {
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] += partials[((int64_t)(p + NG * u) * K + k) * H + col];
    }
    for (; p < P; p += NG) q[0] += partials[((int64_t)p * K + k) * H + col];
    part = (q[0] + q[1]) + (q[2] + q[3]);
  }
  sm[grp][c] = part;
  __syncthreads();
  if (grp != 0 || col >= H) return;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NG; ++i) s += sm[i][c];
  if (out_f32) {
    float* f = reinterpret_cast<float*>(o);
    f[col] = accumulate ? f[col] + s : s;
  } else {
    bf16* b = reinterpret_cast<bf16*>(o);
    b[col] = f2bf(accumulate ? bf2f(b[col]) + s : s);
  }
}

static void colsum_reduce_launch(dim3 grid, const float* partials, int P, int K, int H, void* o0, void* o1, void* o2,
                                 int out_f32, int accumulate, cudaStream_t st) {
  if (P >= 64)
    launch_pdl(colsum_reduce_kernel<32>, grid, 1024, 0, st, partials, P, K, H, o0, o1, o2, out_f32, accumulate);
  else
    launch_pdl(colsum_reduce_kernel<8>, grid, 256, 0, st, partials, P, K, H, o0, o1, o2, out_f32, accumulate);
}

// generic column partial sums of a [M, N] bf16 matrix: grid.x = column blocks of 256, grid.y = row chunks
__global__ void colsum_partial_kernel(const bf16* x, int M, int N, int64_t ldx, int rows_per_chunk, float* partials) {
  pdl_trigger();
  pdl_wait();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= N) return;
  const int r0 = blockIdx.y * rows_per_chunk;
  const int r1 = min(M, r0 + rows_per_chunk);
  float s = 0.f;
  for (int r = r0; r < r1; ++r) s += bf2f(x[(int64_t)r * ldx + col]);
  partials[(int64_t)blockIdx.y * N + col] = s;
}

// ===========================================================================
// softmax forward / backward over attention scores
// ===========================================================================
struct SoftmaxArgs {
  const bf16* s;    // fwd: scores        bwd: probs P
  const bf16* d;    // bwd: dPd (grad of dropped probs)
  bf16* p_out;      // fwd: P             bwd: dS
  bf16* pd_out;     // fwd: dropped probs (p > 0)
  const float* mask;  // [B, s_k] additive, may be null
  int B, nh, sq, sk;
  float scale, p;
  int causal;
  uint64_t seed;
  uint32_t layer;
  int64_t sample_offset;
  int head_offset, nh_global;
  const uint64_t* rng_step = nullptr;
};

__device__ __forceinline__ uint64_t attn_logical_row(const SoftmaxArgs& a, int64_t row) {
  const int64_t q = row % a.sq;
  const int64_t bh = row / a.sq;
  const int64_t h = bh % a.nh;
  const int64_t b = bh / a.nh;
  return (uint64_t)(((a.sample_offset + b) * a.nh_global + a.head_offset + h) * a.sq + q);
}

template <int NV>
__global__ void __launch_bounds__(ROW_THREADS) softmax_fwd_kernel(const SoftmaxArgs a) {
  const uint64_t pkey = philox_key(a.seed, a.rng_step);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)a.B * a.nh * a.sq;
  const float inv_keep = a.p > 0.f ? 1.f / (1.f - a.p) : 1.f;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < rows; row += (int64_t)gridDim.x * 8) {
    const int64_t q = row % a.sq;
    const int64_t b = row / ((int64_t)a.nh * a.sq);
    const int64_t lim = a.causal ? q + (a.sk - a.sq) : (int64_t)a.sk - 1;  // last visible key
    const bf16* src = a.s + row * a.sk;
    float v[NV][8];
    float m = -INFINITY;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int col = (i * 32 + lane) * 8;
      if (col < a.sk) {
        load8(src + col, v[i]);
        float mk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (a.mask) {
          const float4* mp = reinterpret_cast<const float4*>(a.mask + b * a.sk + col);
          float4 m0 = mp[0], m1 = mp[1];
          mk[0] = m0.x; mk[1] = m0.y; mk[2] = m0.z; mk[3] = m0.w;
          mk[4] = m1.x; mk[5] = m1.y; mk[6] = m1.z; mk[7] = m1.w;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float t = v[i][j] * a.scale + mk[j];
          v[i][j] = (col + j > lim) ? -INFINITY : t;
          m = fmaxf(m, v[i][j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[i][j] = -INFINITY;
      }
    }
    m = warp_max(m);
    const float msafe = (m == -INFINITY) ? 0.f : m;
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[i][j] = __expf(v[i][j] - msafe);
        sum += v[i][j];
      }
    sum = warp_sum(sum);
    const float inv = sum > 0.f ? 1.f / sum : 0.f;
    const uint64_t g = a.p > 0.f ? attn_logical_row(a, row) : 0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int col = (i * 32 + lane) * 8;
      if (col < a.sk) {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[i][j] *= inv;
        store8(a.p_out + row * a.sk + col, v[i]);
        if (a.p > 0.f) {
          bool keep[8];
          dropout_keep8(pkey, a.layer, 0u, g, col, dropout_threshold(a.p), keep);
          float o[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] = keep[j] ? round_bf16(v[i][j]) * inv_keep : 0.f;
          store8(a.pd_out + row * a.sk + col, o);
        }
      }
    }
  }
}

template <int NV>
__global__ void __launch_bounds__(ROW_THREADS) softmax_bwd_kernel(const SoftmaxArgs a) {
  const uint64_t pkey = philox_key(a.seed, a.rng_step);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)a.B * a.nh * a.sq;
  const float inv_keep = a.p > 0.f ? 1.f / (1.f - a.p) : 1.f;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < rows; row += (int64_t)gridDim.x * 8) {
    const uint64_t g = a.p > 0.f ? attn_logical_row(a, row) : 0;
    float pv[NV][8], dv[NV][8], pdv[NV][8];
    float c = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int col = (i * 32 + lane) * 8;
      if (col < a.sk) {
        load8(a.s + row * a.sk + col, pv[i]);
        load8(a.d + row * a.sk + col, dv[i]);
        bool keep[8];
        if (a.p > 0.f) {
          dropout_keep8(pkey, a.layer, 0u, g, col, dropout_threshold(a.p), keep);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) keep[j] = true;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          pdv[i][j] = keep[j] ? pv[i][j] * inv_keep : 0.f;
          c += pdv[i][j] * dv[i][j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) pv[i][j] = dv[i][j] = pdv[i][j] = 0.f;
      }
    }
    c = warp_sum(c);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int col = (i * 32 + lane) * 8;
      if (col < a.sk) {
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = a.scale * (pdv[i][j] * dv[i][j] - pv[i][j] * c);
        store8(a.p_out + row * a.sk + col, o);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// dispatch helpers
// ---------------------------------------------------------------------------
#define SMPK_UNPACK(...) __VA_ARGS__
#define SMPK_ROW_CASE(W_, V_, KERNEL, CFG, ARGS) \
  case W_ * 16 + V_:                             \
    launch_pdl(KERNEL<W_, V_>, SMPK_UNPACK CFG, SMPK_UNPACK ARGS); \
    break;
#define SMPK_DISPATCH_ROW(W_, VPT_, KERNEL, CFG, ARGS)                                                  \
  switch ((W_) * 16 + (VPT_)) {                                                                       \
    SMPK_ROW_CASE(1, 1, KERNEL, CFG, ARGS) SMPK_ROW_CASE(1, 2, KERNEL, CFG, ARGS)                      \
    SMPK_ROW_CASE(1, 3, KERNEL, CFG, ARGS) SMPK_ROW_CASE(1, 4, KERNEL, CFG, ARGS)                      \
    SMPK_ROW_CASE(1, 5, KERNEL, CFG, ARGS) SMPK_ROW_CASE(2, 3, KERNEL, CFG, ARGS)                      \
    SMPK_ROW_CASE(2, 4, KERNEL, CFG, ARGS) SMPK_ROW_CASE(2, 5, KERNEL, CFG, ARGS)                      \
    SMPK_ROW_CASE(4, 3, KERNEL, CFG, ARGS) SMPK_ROW_CASE(4, 4, KERNEL, CFG, ARGS)                      \
    SMPK_ROW_CASE(4, 5, KERNEL, CFG, ARGS) SMPK_ROW_CASE(8, 3, KERNEL, CFG, ARGS)                      \
    SMPK_ROW_CASE(8, 4, KERNEL, CFG, ARGS) SMPK_ROW_CASE(8, 5, KERNEL, CFG, ARGS)                      \
    SMPK_ROW_CASE(8, 6, KERNEL, CFG, ARGS) SMPK_ROW_CASE(8, 7, KERNEL, CFG, ARGS)                      \
    SMPK_ROW_CASE(8, 8, KERNEL, CFG, ARGS) SMPK_ROW_CASE(2, 2, KERNEL, CFG, ARGS)                      \
    SMPK_ROW_CASE(4, 2, KERNEL, CFG, ARGS) SMPK_ROW_CASE(8, 2, KERNEL, CFG, ARGS)                      \
    default:                                                                                          \
      set_last_error("unsupported row geometry W=%d VPT=%d", W_, VPT_);                               \
      return SMPK_ERR_UNSUPPORTED;                                                                    \
  }

static bool geom_supported(const RowGeom& g) {
  switch (g.W * 16 + g.VPT) {
    case 17: case 18: case 19: case 20: case 21: case 35: case 36: case 37: case 67: case 68: case 69:
    case 131: case 132: case 133: case 134: case 135: case 136: case 34: case 66: case 130:
      return true;
    default:
      return false;
  }
}

static int softmax_nv(int sk) {
  int need = (sk + 255) / 256;
  if (need <= 1) return 1;
  if (need <= 2) return 2;
  if (need <= 4) return 4;
  if (need <= 8) return 8;
  if (need <= 16) return 16;
  return -1;
}


// ===========================================================================
// Pipelined bias + dropout + residual + LayerNorm (the fast path of smpk_bdr_ln_fwd)
// ===========================================================================
// Persistent CTAs (one per SM).  Warp 0 streams whole input rows into a deep shared-memory
// ring with cp.async.bulk (every partial slot -- local or a peer's over NVLink -- plus the
// residual), so each SM keeps ~100+ KB of row data in flight; 8 consumer warps each own a row
// (lane = 4 x 8-column chunks at H=1024), reduce with warp shuffles only, store r / y locally
// and push y to the peers' gather buffers with bulk shared->global copies.
constexpr int PIPE_CW = 8;  // consumer warps

struct BdrPipeArgs {
  const bf16* x;
  int64_t slot_stride;
  const bf16* const* x_peers;
  int64_t x_peer_off;
  int nslots;
  const bf16* bias;
  const bf16* residual;
  bf16* r_out;
  const bf16* gamma;
  const bf16* beta;
  bf16* y_out;
  float* mean;
  float* rstd;
  int M, H;
  float eps, p;
  uint64_t seed;
  uint32_t layer, site;
  int64_t row_offset;
  uint8_t* keep_out;
  bf16* const* out_peers;  // host-built table copied to the kernel params (<= 8)
  int npeers;
  int64_t peer_off;
  int nst;  // ring stages
  const uint64_t* rng_step = nullptr;
  int push_lsu = 0;  // push the output rows with vector stores instead of bulk copies (SMPK_PIPE_PUSH=lsu)
};

__device__ __forceinline__ void bulk_store_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(gdst)),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}

template <int CH>
__global__ void __launch_bounds__(32 * (PIPE_CW + 1), 1) bdr_ln_pipe_kernel(const BdrPipeArgs a) {
  pdl_trigger();
  pdl_wait();
  const uint64_t pkey = philox_key(a.seed, a.rng_step);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);  // keeps LDS / STS
  const int H = a.H;
  const int nin = a.nslots + (a.residual ? 1 : 0);
  const int stage_bytes = nin * H * 2;
  // per-column parameters (bias | gamma | beta) staged once per CTA
  bf16* par = reinterpret_cast<bf16*>(smem + a.nst * stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.nst * stage_bytes + 3 * H * 2);
  uint64_t* empty = full + a.nst;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
    const uint4 z = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(par + i) = a.bias ? *reinterpret_cast<const uint4*>(a.bias + i) : z;
    *reinterpret_cast<uint4*>(par + H + i) = a.gamma ? *reinterpret_cast<const uint4*>(a.gamma + i) : z;
    *reinterpret_cast<uint4*>(par + 2 * H + i) = a.gamma ? *reinterpret_cast<const uint4*>(a.beta + i) : z;
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int row = blockIdx.x; row < a.M; row += gridDim.x, ++it) {
        const int st = it % a.nst;
        mbar_wait(&empty[st], ((it / a.nst) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], stage_bytes);
        uint8_t* dst = smem + st * stage_bytes;
        for (int j = 0; j < a.nslots; ++j) {
          const bf16* src = a.x_peers ? a.x_peers[j] + a.x_peer_off + (int64_t)row * H
                                      : a.x + j * a.slot_stride + (int64_t)row * H;
          bulk_load(dst + j * H * 2, src, H * 2, &full[st]);
        }
        if (a.residual) bulk_load(dst + a.nslots * H * 2, a.residual + (int64_t)row * H, H * 2, &full[st]);
      }
    }
    return;
  }
  // ---------------- consumers: warp c handles iterations it == c (mod PIPE_CW) ----------------
  const int c = warp - 1;
  const float inv_keep = a.p > 0.f ? 1.f / (1.f - a.p) : 1.f;
  const uint32_t thresh = dropout_threshold(a.p);
  int it = c;
  for (int row = blockIdx.x + c * gridDim.x; row < a.M; row += PIPE_CW * gridDim.x, it += PIPE_CW) {
    const int st = it % a.nst;
    mbar_wait(&full[st], (it / a.nst) & 1);
    const uint8_t* buf = smem + st * stage_bytes;
    float v[CH][8];
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int col = (k * 32 + lane) * 8;
      load8(reinterpret_cast<const bf16*>(buf) + col, v[k]);
      for (int j = 1; j < a.nslots; ++j) {  // ascending rank order
        float t[8];
        load8(reinterpret_cast<const bf16*>(buf + j * H * 2) + col, t);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[k][e] += t[e];
      }
      if (a.bias) {
        float bv[8];
        load8(par + col, bv);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[k][e] += bv[e];
      }
      if (a.p > 0.f) {
        bool keep[8];
        dropout_keep8(pkey, a.layer, a.site, (uint64_t)(a.row_offset + row), col, thresh, keep);
        if (a.keep_out) a.keep_out[(int64_t)row * (H / 8) + col / 8] = (uint8_t)keep8_to_byte(keep);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[k][e] = keep[e] ? v[k][e] * inv_keep : 0.f;
      }
      if (a.residual) {
        float rr[8];
        load8(reinterpret_cast<const bf16*>(buf + a.nslots * H * 2) + col, rr);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[k][e] += rr[e];
      }
      round8(v[k]);
    }
    __syncwarp();
    const bool push = a.npeers > 0 && !a.push_lsu;  // bulk push from the stage
    if (!push) {
      if (lane == 0) mbar_arrive(&empty[st]);  // inputs consumed: the producer may refill
    }
    if (a.r_out) {
#pragma unroll
      for (int k = 0; k < CH; ++k) store8(a.r_out + (int64_t)row * H + (k * 32 + lane) * 8, v[k]);
    }
    float o[CH][8];
    if (a.gamma) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < CH; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) s += v[k][e];
      const float mu = warp_sum(s) / H;
      float q = 0.f;
#pragma unroll
      for (int k = 0; k < CH; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = v[k][e] - mu;
          q += d * d;
        }
      const float rs = rsqrtf(warp_sum(q) / H + a.eps);
      if (lane == 0) {
        a.mean[row] = mu;
        a.rstd[row] = rs;
      }
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        float gv[8], bv[8];
        load8(par + H + (k * 32 + lane) * 8, gv);
        load8(par + 2 * H + (k * 32 + lane) * 8, bv);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[k][e] = (v[k][e] - mu) * rs * gv[e] + bv[e];
      }
      if (a.y_out) {
#pragma unroll
        for (int k = 0; k < CH; ++k) store8(a.y_out + (int64_t)row * H + (k * 32 + lane) * 8, o[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < CH; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) o[k][e] = v[k][e];
    }
    if (a.npeers && a.push_lsu) {  // push with plain vector stores (LSU path, next to the TMA pulls)
#pragma unroll
      for (int k = 0; k < CH; ++k)
        store8_peers(a.out_peers, a.npeers, a.peer_off + (int64_t)row * H + (k * 32 + lane) * 8, o[k]);
    }
    if (push) {
      // the stage's first slot row becomes the bf16 output row, pushed to every peer in bulk
      bf16* obuf = reinterpret_cast<bf16*>(smem + st * stage_bytes);
#pragma unroll
      for (int k = 0; k < CH; ++k) store8(obuf + (k * 32 + lane) * 8, o[k]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        for (int j = 0; j < a.npeers; ++j)
          bulk_store_s2g(a.out_peers[j] + a.peer_off + (int64_t)row * H, obuf, H * 2);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbar_arrive(&empty[st]);
      }
      __syncwarp();
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static int bdr_ln_pipe_launch(const BdrPipeArgs& a, cudaStream_t st) {
  const int nin = a.nslots + (a.residual ? 1 : 0);
  const int stage_bytes = nin * a.H * 2;
  const int smem = a.nst * stage_bytes + 3 * a.H * 2 + 2 * a.nst * 8 + 128;
  const int grid = a.M < row_sms() ? a.M : row_sms();
  switch (a.H / 256) {
#define SMPK_PIPE_CASE(CH_)                                                                              \
  case CH_: {                                                                                            \
    static unsigned long long once = 0;                                                                  \
    smem_attr_once(bdr_ln_pipe_kernel<CH_>, 232448, once);                                               \
    launch_pdl(bdr_ln_pipe_kernel<CH_>, grid, 32 * (PIPE_CW + 1), smem, st, a);                           \
    break;                                                                                               \
  }
    SMPK_PIPE_CASE(1) SMPK_PIPE_CASE(2) SMPK_PIPE_CASE(4) SMPK_PIPE_CASE(8)
#undef SMPK_PIPE_CASE
    default:
      return SMPK_ERR_UNSUPPORTED;
  }
  return check_launch("smpk_bdr_ln_fwd(pipe)");
}

}  // namespace smpk

using namespace smpk;

// SMPK_ROW_PIPE=0 selects the register-only row kernel (A/B measurements)
// SMPK_ROW_PIPE_LOCAL=1 routes local-row bias/dropout/residual/LayerNorm calls through the pipelined
// kernel too (A/B measurements)
static bool pipe_local() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMPK_ROW_PIPE_LOCAL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

static bool push_lsu_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMPK_PIPE_PUSH");
    v = (e && e[0] == 'l') ? 1 : 0;
  }
  return v == 1;
}

static bool pipe_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMPK_ROW_PIPE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <bool BR, bool LN>
static int launch_fast(const RowGeom& geo, int grid, cudaStream_t st, const BdrLnArgs& a) {
  switch (geo.W * 16 + geo.VPT) {
    case 17: launch_pdl(bdr_ln_fwd_fast_kernel<1, 1, BR, LN>, grid, ROW_THREADS, 0, st, a); return 0;
    case 18: launch_pdl(bdr_ln_fwd_fast_kernel<1, 2, BR, LN>, grid, ROW_THREADS, 0, st, a); return 0;
    case 34: launch_pdl(bdr_ln_fwd_fast_kernel<2, 2, BR, LN>, grid, ROW_THREADS, 0, st, a); return 0;
    case 66: launch_pdl(bdr_ln_fwd_fast_kernel<4, 2, BR, LN>, grid, ROW_THREADS, 0, st, a); return 0;
    case 130: launch_pdl(bdr_ln_fwd_fast_kernel<8, 2, BR, LN>, grid, ROW_THREADS, 0, st, a); return 0;
    default: return -1;
  }
}

static int bdr_ln_impl(const void* x, int nslots, int64_t slot_stride, const void* bias, const void* residual,
                       void* r_out, const void* gamma, const void* beta, void* y_out, float* mean, float* rstd,
                       void* const* out_peers, int npeers, int64_t peer_off, int M, int H, float eps, float p_drop,
                       uint64_t seed, const uint64_t* rng_step, int layer, int site, int64_t row_offset,
                       int64_t col_offset, float* row_sums_out, const float* ext_sums, int H_total,
                       uint8_t* keep_out, void* const* x_peers, int64_t x_peer_off, void* stream) {
  RowGeom geo;
  SMPK_REQUIRE(M >= 0 && row_geom(H, geo) && geom_supported(geo), SMPK_ERR_UNSUPPORTED,
               "smpk_bdr_ln_fwd: hidden size %d unsupported (need a multiple of 8)", H);
  SMPK_REQUIRE((x != nullptr || x_peers != nullptr) && nslots >= 1, SMPK_ERR_BAD_ARG, "smpk_bdr_ln_fwd: null x");
  SMPK_REQUIRE(!x_peers || nslots <= 8, SMPK_ERR_UNSUPPORTED, "smpk_bdr_ln_fwd: at most 8 peer slots");
  SMPK_REQUIRE(gamma == nullptr || (beta && mean && rstd && (y_out || npeers)), SMPK_ERR_BAD_ARG,
               "smpk_bdr_ln_fwd: LayerNorm needs beta, mean, rstd and an output");
  SMPK_REQUIRE(gamma != nullptr || r_out != nullptr || npeers > 0 || row_sums_out, SMPK_ERR_BAD_ARG,
               "smpk_bdr_ln_fwd: nothing to compute");
  SMPK_REQUIRE(!ext_sums || H_total > 0, SMPK_ERR_BAD_ARG, "smpk_bdr_ln_fwd_dist: H_total must be positive");
  SMPK_REQUIRE(npeers == 0 || out_peers != nullptr, SMPK_ERR_BAD_ARG, "smpk_bdr_ln_fwd: null peer table");
  SMPK_REQUIRE(p_drop >= 0.f && p_drop < 1.f, SMPK_ERR_BAD_ARG, "smpk_bdr_ln_fwd: dropout p must be in [0,1)");
  if (M == 0) return SMPK_OK;
  BdrLnArgs a{reinterpret_cast<const bf16*>(x), reinterpret_cast<const bf16*>(bias),
              reinterpret_cast<const bf16*>(residual), reinterpret_cast<bf16*>(r_out),
              reinterpret_cast<const bf16*>(gamma), reinterpret_cast<const bf16*>(beta),
              reinterpret_cast<bf16*>(y_out), mean, rstd, M, H, eps, p_drop, seed, (uint32_t)layer, (uint32_t)site,
              row_offset, nslots, slot_stride, reinterpret_cast<bf16* const*>(out_peers), npeers, peer_off,
              col_offset, row_sums_out, ext_sums, H_total, keep_out, reinterpret_cast<const bf16* const*>(x_peers),
              x_peer_off};
  a.rng_step = rng_step;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // pipelined path for the TP exchanges (partials pulled from peers and/or output pushed to peers:
  // bulk copies keep enough NVLink traffic in flight); whole 16-B aligned rows, <= 2048 columns.
  // Purely local rows stay on the register kernel below (measured faster for them).
  const int ch = H / 256;
  const bool al = (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(residual) |
                   reinterpret_cast<uintptr_t>(r_out) | reinterpret_cast<uintptr_t>(y_out)) % 16 == 0 &&
                  (slot_stride * 2) % 16 == 0 && (x_peer_off * 2) % 16 == 0 && (peer_off * 2) % 16 == 0;
  if (pipe_enabled() && (x_peers || npeers || pipe_local()) && H % 256 == 0 && (ch == 1 || ch == 2 || ch == 4 || ch == 8) && al &&
      !row_sums_out &&
      !ext_sums && col_offset == 0 && nslots <= 8 && npeers <= 8) {
    BdrPipeArgs pa{reinterpret_cast<const bf16*>(x), slot_stride, reinterpret_cast<const bf16* const*>(x_peers),
                   x_peer_off, nslots, reinterpret_cast<const bf16*>(bias), reinterpret_cast<const bf16*>(residual),
                   reinterpret_cast<bf16*>(r_out), reinterpret_cast<const bf16*>(gamma),
                   reinterpret_cast<const bf16*>(beta), reinterpret_cast<bf16*>(y_out), mean, rstd, M, H, eps,
                   p_drop, seed, (uint32_t)layer, (uint32_t)site, row_offset, keep_out,
                   reinterpret_cast<bf16* const*>(out_peers), npeers, peer_off, 0};
  pa.rng_step = rng_step;
  pa.push_lsu = push_lsu_enabled() ? 1 : 0;
    const int nin = nslots + (residual ? 1 : 0);
    const int budget = 200 * 1024 - 3 * H * 2;
    const int nst = budget / (nin * H * 2);
    // consumer warp c owns the iterations it == c (mod PIPE_CW) and reads stage it % nst: with nst a
    // multiple of PIPE_CW every stage has exactly one owning warp, so a warp can never wait on a
    // stage phase that another warp's row is still filling or reading (nst = 5 / 9 / 10
    // aliased stages across warps).  Fewer than PIPE_CW stages fit: use the register kernel.
    pa.nst = ((nst > 16 ? 16 : nst) / PIPE_CW) * PIPE_CW;
    if (pa.nst >= PIPE_CW) return bdr_ln_pipe_launch(pa, st);
  }
  // 80 registers with the next-row prefetch: 3 resident CTAs per SM, one wave
  const int grid = row_grid(M, geo.W, 3);
  if (fast_enabled() && !x_peers && nslots == 1 && npeers == 0 && !row_sums_out && !ext_sums && col_offset == 0 &&
      H == geo.W * geo.VPT * 256 && !(reinterpret_cast<uintptr_t>(x) & 15) && geo.VPT <= 2 &&
      (geo.W == 1 || geo.W == 2 || geo.W == 4 || geo.W == 8)) {
    const bool br = bias && residual, ln = gamma && y_out;
    int rc = -1;
    if (br && ln) rc = launch_fast<true, true>(geo, grid, st, a);
    else if (br && !gamma && r_out) rc = launch_fast<true, false>(geo, grid, st, a);
    else if (!bias && !residual && p_drop == 0.f && !keep_out && ln) rc = launch_fast<false, true>(geo, grid, st, a);
    if (rc >= 0) return check_launch("smpk_bdr_ln_fwd(fast)");
  }
  SMPK_DISPATCH_ROW(geo.W, geo.VPT, bdr_ln_fwd_kernel, (grid, ROW_THREADS, 0, st), (a));
  return check_launch("smpk_bdr_ln_fwd");
}

extern "C" int smpk_bdr_ln_fwd_ex(const void* x, int nslots, int64_t slot_stride, const void* bias,
                                  const void* residual, void* r_out, const void* gamma, const void* beta, void* y_out,
                                  float* mean, float* rstd, void* const* out_peers, int npeers, int64_t peer_off, int M,
                                  int H, float eps, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer, int site,
                                  int64_t row_offset, void* keep_out, void* const* x_peers, int64_t x_peer_off,
                                  void* stream) {
  return bdr_ln_impl(x, nslots, slot_stride, bias, residual, r_out, gamma, beta, y_out, mean, rstd, out_peers, npeers,
                     peer_off, M, H, eps, p_drop, seed, rng_step, layer, site, row_offset, 0, nullptr, nullptr, 0,
                     reinterpret_cast<uint8_t*>(keep_out), x_peers, x_peer_off, stream);
}

extern "C" int smpk_bdr_ln_fwd_dist(const void* x, const void* bias, const void* residual, void* r_out,
                                    const void* gamma, const void* beta, void* y_out, float* mean, float* rstd,
                                    int M, int H, float eps, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer, int site,
                                    int64_t row_offset, int64_t col_offset, float* row_sums_out,
                                    const float* ext_sums, int H_total, void* stream) {
  return bdr_ln_impl(x, 1, 0, bias, residual, r_out, gamma, beta, y_out, mean, rstd, nullptr, 0, 0, M, H, eps, p_drop,
                     seed, rng_step, layer, site, row_offset, col_offset, row_sums_out, ext_sums, H_total, nullptr, nullptr, 0,
                     stream);
}

extern "C" int smpk_bdr_ln_fwd(const void* x, const void* bias, const void* residual, void* r_out, const void* gamma,
                               const void* beta, void* y_out, float* mean, float* rstd, int M, int H, float eps,
                               float p_drop, uint64_t seed, const uint64_t* rng_step, int layer, int site, int64_t row_offset, void* stream) {
  return smpk_bdr_ln_fwd_ex(x, 1, 0, bias, residual, r_out, gamma, beta, y_out, mean, rstd, nullptr, 0, 0, M, H, eps,
                            p_drop, seed, rng_step, layer, site, row_offset, nullptr, nullptr, 0, stream);
}

// The backward keeps per-column accumulators in registers (two CTAs per SM): one wave of
// 2 x #SM persistent CTAs, each flushing its column partials once.
static int ln_bwd_grid_geo(int M, int W) {
  const int rows_per_cta = (ROW_THREADS / 32) / W;
  const int need = (M + rows_per_cta - 1) / rows_per_cta;
  const int cap = 2 * row_sms();
  return need < cap ? need : cap;
}

static int64_t ln_bwd_grid(int M, int H) {
  RowGeom geo;
  if (!row_geom(H, geo)) return 0;
  return ln_bwd_grid_geo(M, geo.W);
}

extern "C" int64_t smpk_ln_bwd_workspace(int M, int H) { return ln_bwd_grid(M, H) * 3 * (int64_t)H * 4; }


// ===========================================================================
// Pipelined LayerNorm / dropout backward (local rows): the fast path of smpk_ln_bwd
// ===========================================================================
// One persistent CTA per SM.  Warp 0 streams each row's inputs (dy, r, dres, keep bytes) into a
// deep shared-memory ring with cp.async.bulk, so ~150-200 KB of rows are in flight per SM instead
// of the few rows the register kernel holds; 16 consumer warps form groups of W warps (one row
// per group at a time, the lane layout and column accumulators of ln_bwd_kernel), read their
// row from shared memory, and the groups' column partials are summed in ascending group order
// (deterministic) into this CTA's partial row of the workspace.
// consumer warps: 12 (13 warps allocate registers like 16 -> 128 per thread, no spills), 8 at W = 8
__host__ __device__ constexpr int lnb_cw(int W) { return W == 8 ? 8 : 12; }

template <int W>
__device__ __forceinline__ void group_bar(int grp) {
  if constexpr (W > 1) named_bar(1 + grp, W * 32);
  else __syncwarp();
}

template <int W, int VPT>
__global__ void __launch_bounds__(32 * (lnb_cw(W) + 1), 1) ln_bwd_pipe_kernel(const LnBwdArgs a, int nst, int sb) {
  pdl_trigger();
  pdl_wait();
  constexpr int LNB_CW = lnb_cw(W);
  constexpr int G = LNB_CW / W;  // row groups
  const uint64_t pkey = philox_key(a.seed, a.rng_step);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  const int H = a.H;
  const bool has_ln = a.gamma != nullptr;
  const int o_r = H * 2, o_dres = o_r + (has_ln ? H * 2 : 0), o_keep = o_dres + (a.dres ? H * 2 : 0);
  const int in_bytes = o_keep + (a.keep_in ? H / 8 : 0);
  float* red = reinterpret_cast<float*>(smem + nst * sb);  // [W][VPT*8][32] flush buffer
  float* sm = red + W * VPT * 8 * 32;                        // [2][LNB_CW] group sums
  bf16* gam = reinterpret_cast<bf16*>(sm + 2 * LNB_CW);     // gamma [H]
  uint64_t* full = reinterpret_cast<uint64_t*>(gam + H);
  uint64_t* empty = full + nst;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], W);  // every warp of the owning group releases it
    }
    fence_barrier_init();
  }
  if (has_ln)
    for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8)
      *reinterpret_cast<uint4*>(gam + i) = *reinterpret_cast<const uint4*>(a.gamma + i);
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int row = blockIdx.x; row < a.M; row += gridDim.x, ++it) {
        const int st = it % nst;
        mbar_wait(&empty[st], ((it / nst) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], in_bytes);
        uint8_t* dst = smem + st * sb;
        const int64_t ro = (int64_t)row * H;
        bulk_load(dst, a.dy + ro, H * 2, &full[st]);
        if (has_ln) bulk_load(dst + o_r, a.r + ro, H * 2, &full[st]);
        if (a.dres) bulk_load(dst + o_dres, a.dres + ro, H * 2, &full[st]);
        if (a.keep_in) bulk_load(dst + o_keep, a.keep_in + (int64_t)row * (H / 8), H / 8, &full[st]);
      }
    }
    return;
  }
  const int c = warp - 1, grp = c / W, wi = c % W;
  const float inv_keep = a.p > 0.f ? 1.f / (1.f - a.p) : 1.f;
  const float inv_h = 1.f / H;
  // paired fp32 math (FFMA2 / FADD2 / FMUL2) on (even, odd) column pairs
  float2 acc_g[VPT][4], acc_b[VPT][4], acc_d[VPT][4];
#pragma unroll
  for (int i = 0; i < VPT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc_g[i][j] = acc_b[i][j] = acc_d[i][j] = make_float2(0.f, 0.f);
  const float2 ik2 = make_float2(inv_keep, inv_keep);
  int it = grp;
  for (int row = blockIdx.x + grp * gridDim.x; row < a.M; row += G * gridDim.x, it += G) {
    const int st = it % nst;
    const float mu = has_ln ? a.mean[row] : 0.f, rs = has_ln ? a.rstd[row] : 0.f;
    const float2 nmu2 = make_float2(-mu, -mu), rs2 = make_float2(rs, rs);
    mbar_wait(&full[st], (it / nst) & 1);
    const uint8_t* buf = smem + st * sb;
    // pass 1 (LayerNorm): row sums of g = dy*gamma and g*xhat, column sums of dy*xhat and dy
    float2 nm1 = make_float2(0.f, 0.f), nm2 = make_float2(0.f, 0.f);
    if (has_ln) {
      float2 s1 = make_float2(0.f, 0.f), s2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int col = ((i * W + wi) * 32 + lane) * 8;
        const uint4 du = *reinterpret_cast<const uint4*>(buf + col * 2);
        const uint4 ru = *reinterpret_cast<const uint4*>(buf + o_r + col * 2);
        const uint4 gu = *reinterpret_cast<const uint4*>(gam + col);
        const uint32_t dw[4] = {du.x, du.y, du.z, du.w}, rw[4] = {ru.x, ru.y, ru.z, ru.w},
                       gw[4] = {gu.x, gu.y, gu.z, gu.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 dy = unpack_bf16x2(dw[j]);
          const float2 xh = __fmul2_rn(__fadd2_rn(unpack_bf16x2(rw[j]), nmu2), rs2);
          const float2 gj = __fmul2_rn(dy, unpack_bf16x2(gw[j]));
          s1 = __fadd2_rn(s1, gj);
          s2 = __ffma2_rn(gj, xh, s2);
          acc_g[i][j] = __ffma2_rn(dy, xh, acc_g[i][j]);
          acc_b[i][j] = __fadd2_rn(acc_b[i][j], dy);
        }
      }
      const float2 m = group_sum2<W>(make_float2(s1.x + s1.y, s2.x + s2.y), sm, grp, wi);
      nm1 = make_float2(-m.x * inv_h, -m.x * inv_h);
      nm2 = make_float2(-m.y * inv_h, -m.y * inv_h);
    }
    // pass 2: d = rs*(g - m1 - xhat*m2) (+ dres), dropout backward, stores (inputs re-read from smem)
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int col = ((i * W + wi) * 32 + lane) * 8;
      const uint4 du = *reinterpret_cast<const uint4*>(buf + col * 2);
      const uint32_t dw[4] = {du.x, du.y, du.z, du.w};
      float2 d[4];
      if (has_ln) {
        const uint4 ru = *reinterpret_cast<const uint4*>(buf + o_r + col * 2);
        const uint4 gu = *reinterpret_cast<const uint4*>(gam + col);
        const uint32_t rw[4] = {ru.x, ru.y, ru.z, ru.w}, gw[4] = {gu.x, gu.y, gu.z, gu.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 xh = __fmul2_rn(__fadd2_rn(unpack_bf16x2(rw[j]), nmu2), rs2);
          const float2 u = __ffma2_rn(unpack_bf16x2(dw[j]), unpack_bf16x2(gw[j]), nm1);
          d[j] = __fmul2_rn(__ffma2_rn(xh, nm2, u), rs2);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) d[j] = unpack_bf16x2(dw[j]);
      }
      if (a.dres) {
        const uint4 eu = *reinterpret_cast<const uint4*>(buf + o_dres + col * 2);
        const uint32_t ew[4] = {eu.x, eu.y, eu.z, eu.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) d[j] = __fadd2_rn(d[j], unpack_bf16x2(ew[j]));
      }
      uint32_t pk[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        pk[j] = pack_bf16x2(d[j].x, d[j].y);  // dr in bf16
        d[j] = unpack_bf16x2(pk[j]);
      }
      if (a.dr_out) *reinterpret_cast<uint4*>(a.dr_out + (int64_t)row * H + col) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      if (a.p > 0.f) {
        bool keep[8];
        if (a.keep_in)
          keep8_from_byte(buf[o_keep + col / 8], keep);
        else
          dropout_keep8(pkey, a.layer, a.site, (uint64_t)(a.row_offset + row), col, dropout_threshold(a.p), keep);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 t = __fmul2_rn(d[j], ik2);
          t.x = keep[2 * j] ? t.x : 0.f;
          t.y = keep[2 * j + 1] ? t.y : 0.f;
          pk[j] = pack_bf16x2(t.x, t.y);  // dsub in bf16
          d[j] = unpack_bf16x2(pk[j]);
        }
        *reinterpret_cast<uint4*>(a.dsub_out + (int64_t)row * H + col) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      if (a.npeers)  // dy slot := output
        *reinterpret_cast<uint4*>(const_cast<uint8_t*>(buf) + col * 2) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
#pragma unroll
      for (int j = 0; j < 4; ++j) acc_d[i][j] = __fadd2_rn(acc_d[i][j], d[j]);
    }
    if (a.npeers) {
      // the row's output (in the stage's dy slot) goes to every peer's gather region in bulk; the
      // stage is released only once the copies have read it
      fence_proxy_async_smem();
      group_bar<W>(grp);
      if (wi == 0 && lane == 0) {
        for (int j = 0; j < a.npeers; ++j)
          bulk_store_s2g(a.out_peers[j] + a.peer_off + (int64_t)row * H, buf, H * 2);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (a.npeers && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // column partials of the CTA: groups summed in ascending order through shared memory
  float* out = a.partials + (int64_t)blockIdx.x * 3 * H;
  float* rbuf = red + wi * (VPT * 8 * 32);
  auto flush = [&](const float2(&acc)[VPT][4], float* o) {
    for (int sl = 0; sl < G; ++sl) {
      if (grp == sl) {
#pragma unroll
        for (int i = 0; i < VPT; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float* dd = rbuf + (i * 8 + j) * 32 + lane;
            const float av = (j & 1) ? acc[i][j >> 1].y : acc[i][j >> 1].x;
            *dd = (sl == 0) ? av : *dd + av;
          }
      }
      named_bar(15, LNB_CW * 32);
    }
    if (grp == G - 1) {
#pragma unroll
      for (int i = 0; i < VPT; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) o[((i * W + wi) * 32 + lane) * 8 + j] = rbuf[(i * 8 + j) * 32 + lane];
    }
    named_bar(15, LNB_CW * 32);
  };
  flush(acc_g, out);
  flush(acc_b, out + H);
  flush(acc_d, out + 2 * H);
}

static bool lnb_pipe_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMPK_LNB_PIPE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// Launches the pipelined backward when the call is a plain local one; returns -1 when it does not apply.
static int ln_bwd_pipe_try(const LnBwdArgs& a, const RowGeom& geo, cudaStream_t st, int grid_limit) {
  if (!lnb_pipe_enabled() || a.npeers > 8 || a.dy_peers || a.nslots != 1 || a.row_sums_out || a.ext_sums ||
      a.col_offset || geo.W < 2 || a.H != geo.W * geo.VPT * 256 || a.M < 1 || (a.peer_off * 2) % 16)
    return -1;
  const uintptr_t al = reinterpret_cast<uintptr_t>(a.dy) | reinterpret_cast<uintptr_t>(a.r) |
                       reinterpret_cast<uintptr_t>(a.dres) | reinterpret_cast<uintptr_t>(a.keep_in) |
                       reinterpret_cast<uintptr_t>(a.dr_out) | reinterpret_cast<uintptr_t>(a.dsub_out);
  if (al % 16) return -1;
  const int H = a.H;
  const int in_bytes = H * 2 + (a.gamma ? H * 2 : 0) + (a.dres ? H * 2 : 0) + (a.keep_in ? H / 8 : 0);
  const int sb = (in_bytes + 127) / 128 * 128;
  const int CW = lnb_cw(geo.W), G = CW / geo.W;
  const int fixed = geo.W * geo.VPT * 8 * 32 * 4 + 2 * CW * 4 + H * 2 + 128;
  int nst = (200 * 1024 - fixed) / (sb + 16);
  if (nst > 48) nst = 48;
  nst = nst / G * G;  // every stage owned by exactly one row group
  if (nst < G) return -1;
  const int smem = nst * sb + fixed + 2 * nst * 8;
  int grid = row_sms();
  if (grid > grid_limit) grid = grid_limit;
  if (grid > a.M) grid = a.M;
  switch (geo.W * 16 + geo.VPT) {
#define SMPK_LNB_CASE(W_, V_)                                                                    \
  case W_ * 16 + V_: {                                                                           \
    static unsigned long long once = 0;                                                          \
    smem_attr_once(ln_bwd_pipe_kernel<W_, V_>, 232448, once);                                    \
    launch_pdl(ln_bwd_pipe_kernel<W_, V_>, grid, 32 * (lnb_cw(W_) + 1), smem, st, a, nst, sb);   \
    return grid;                                                                                 \
  }
    SMPK_LNB_CASE(2, 2) SMPK_LNB_CASE(4, 2) SMPK_LNB_CASE(8, 2) SMPK_LNB_CASE(2, 1) SMPK_LNB_CASE(4, 1)
    SMPK_LNB_CASE(8, 1)
#undef SMPK_LNB_CASE
    default:
      return -1;
  }
}

static int ln_bwd_impl(const void* dy, int nslots, int64_t slot_stride, const void* r, const float* mean,
                       const float* rstd, const void* gamma, const void* dres, void* dr_out, void* dsub_out,
                       void* const* out_peers, int npeers, int64_t peer_off, void* dgamma, void* dbeta, void* dbias,
                       int grads_f32, int accumulate, int M, int H, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer, int site,
                       int64_t row_offset, int64_t col_offset, float* row_sums_out, const float* ext_sums,
                       int H_total, const uint8_t* keep_in, void* const* dy_peers, int64_t dy_peer_off,
                       void* workspace, int64_t workspace_bytes, void* stream) {
  RowGeom geo;
  SMPK_REQUIRE(M > 0 && row_geom(H, geo) && geom_supported(geo), SMPK_ERR_UNSUPPORTED,
               "smpk_ln_bwd: hidden size %d unsupported", H);
  SMPK_REQUIRE(!dy_peers || nslots <= 8, SMPK_ERR_UNSUPPORTED, "smpk_ln_bwd: at most 8 peer slots");
  SMPK_REQUIRE((dy || dy_peers) && nslots >= 1 && (gamma == nullptr || (r && mean && rstd && (dr_out || row_sums_out))),
               SMPK_ERR_BAD_ARG, "smpk_ln_bwd: null argument");
  SMPK_REQUIRE(!row_sums_out || (gamma && !ext_sums), SMPK_ERR_BAD_ARG,
               "smpk_ln_bwd_dist: the sums pass needs gamma and no external sums");
  SMPK_REQUIRE(!ext_sums || H_total > 0, SMPK_ERR_BAD_ARG, "smpk_ln_bwd_dist: H_total must be positive");
  SMPK_REQUIRE(p_drop == 0.f || dsub_out || row_sums_out, SMPK_ERR_BAD_ARG,
               "smpk_ln_bwd: dropout backward needs dsub_out");
  SMPK_REQUIRE(npeers == 0 || out_peers, SMPK_ERR_BAD_ARG, "smpk_ln_bwd: null peer table");
  const int grid = ln_bwd_grid_geo(M, geo.W);
  SMPK_REQUIRE(workspace && workspace_bytes >= (int64_t)grid * 3 * H * 4, SMPK_ERR_BAD_ARG,
               "smpk_ln_bwd: workspace too small (%lld < %lld)", (long long)workspace_bytes,
               (long long)grid * 3 * H * 4);
  LnBwdArgs a{reinterpret_cast<const bf16*>(dy), reinterpret_cast<const bf16*>(r), mean, rstd,
              reinterpret_cast<const bf16*>(gamma), reinterpret_cast<const bf16*>(dres),
              reinterpret_cast<bf16*>(dr_out), reinterpret_cast<bf16*>(dsub_out),
              reinterpret_cast<float*>(workspace), M, H, p_drop, seed, (uint32_t)layer, (uint32_t)site, row_offset,
              nslots, slot_stride, reinterpret_cast<bf16* const*>(out_peers), npeers, peer_off, col_offset,
              row_sums_out, ext_sums, H_total, keep_in, reinterpret_cast<const bf16* const*>(dy_peers), dy_peer_off};
  a.rng_step = rng_step;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int used_grid = ln_bwd_pipe_try(a, geo, st, grid);
  if (used_grid < 0) {
    const int red_bytes = geo.W == 8 ? 0 : geo.W * geo.VPT * 8 * 32 * 4;
    SMPK_DISPATCH_ROW(geo.W, geo.VPT, ln_bwd_kernel, (grid, ROW_THREADS, red_bytes, st), (a));
    used_grid = grid;
  }
  int rc = check_launch("smpk_ln_bwd");
  if (rc) return rc;
  if (row_sums_out || (!dgamma && !dbeta && !dbias)) return SMPK_OK;
  dim3 rg((H + 31) / 32, 3);
  colsum_reduce_launch(rg, reinterpret_cast<float*>(workspace), used_grid, 3, H, dgamma, dbeta, dbias, grads_f32,
                       accumulate, st);
  return check_launch("smpk_ln_bwd(reduce)");
}

extern "C" int smpk_ln_bwd_ex(const void* dy, int nslots, int64_t slot_stride, const void* r, const float* mean,
                              const float* rstd, const void* gamma, const void* dres, void* dr_out, void* dsub_out,
                              void* const* out_peers, int npeers, int64_t peer_off, void* dgamma, void* dbeta,
                              void* dbias, int grads_f32, int accumulate, int M, int H, float p_drop, uint64_t seed, const uint64_t* rng_step,
                              int layer, int site, int64_t row_offset, const void* keep_in, void* const* dy_peers,
                              int64_t dy_peer_off, void* workspace, int64_t workspace_bytes, void* stream) {
  return ln_bwd_impl(dy, nslots, slot_stride, r, mean, rstd, gamma, dres, dr_out, dsub_out, out_peers, npeers,
                     peer_off, dgamma, dbeta, dbias, grads_f32, accumulate, M, H, p_drop, seed, rng_step, layer, site,
                     row_offset, 0, nullptr, nullptr, 0, reinterpret_cast<const uint8_t*>(keep_in), dy_peers,
                     dy_peer_off, workspace, workspace_bytes, stream);
}

extern "C" int smpk_ln_bwd_dist(const void* dy, const void* r, const float* mean, const float* rstd,
                                const void* gamma, const void* dres, void* dr_out, void* dsub_out, void* dgamma,
                                void* dbeta, void* dbias, int grads_f32, int M, int H, float p_drop, uint64_t seed, const uint64_t* rng_step,
                                int layer, int site, int64_t row_offset, int64_t col_offset, float* row_sums_out,
                                const float* ext_sums, int H_total, void* workspace, int64_t workspace_bytes,
                                void* stream) {
  return ln_bwd_impl(dy, 1, 0, r, mean, rstd, gamma, dres, dr_out, dsub_out, nullptr, 0, 0, dgamma, dbeta, dbias,
                     grads_f32, 0, M, H, p_drop, seed, rng_step, layer, site, row_offset, col_offset, row_sums_out, ext_sums,
                     H_total, nullptr, nullptr, 0, workspace, workspace_bytes, stream);
}

extern "C" int smpk_ln_bwd(const void* dy, const void* r, const float* mean, const float* rstd, const void* gamma,
                           const void* dres, void* dr_out, void* dsub_out, void* dgamma, void* dbeta, void* dbias,
                           int grads_f32, int accumulate, int M, int H, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer,
                           int site, int64_t row_offset, void* workspace, int64_t workspace_bytes, void* stream) {
  return smpk_ln_bwd_ex(dy, 1, 0, r, mean, rstd, gamma, dres, dr_out, dsub_out, nullptr, 0, 0, dgamma, dbeta, dbias,
                        grads_f32, accumulate, M, H, p_drop, seed, rng_step, layer, site, row_offset, nullptr, nullptr, 0,
                        workspace, workspace_bytes, stream);
}

// Column sums from fp32 partial rows [P][N] (e.g. the GEMM epilogue's per-box sums), in order.
extern "C" int smpk_colsum_partials(const float* part, int P, int N, void* out, int out_f32, void* stream) {
  SMPK_REQUIRE(part && out && P > 0 && N > 0, SMPK_ERR_BAD_ARG, "smpk_colsum_partials: bad arguments");
  dim3 g2((N + 31) / 32, 1);
  colsum_reduce_launch(g2, part, P, 1, N, out, nullptr, nullptr, out_f32, 0,
                       reinterpret_cast<cudaStream_t>(stream));
  return check_launch("smpk_colsum_partials");
}

// ===========================================================================
// bias + activation (channel-sharded MLP of memory mode: the activation follows a
// reduce-scatter, so it cannot live in the GEMM epilogue)
// ===========================================================================
template <int ACT>
__global__ void __launch_bounds__(256) bias_act_fwd_kernel(const bf16* __restrict__ x, const bf16* __restrict__ bias,
                                                           int64_t n8, int N, bf16* __restrict__ pre,
                                                           bf16* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)((i * 8) % N);
    float v[8], b[8];
    load8(x + i * 8, v);
    load8(bias + col, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = round_bf16(v[j] + b[j]);
    store8(pre + i * 8, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = act_fwd(ACT, v[j]);
    store8(y + i * 8, v);
  }
}

template <int ACT>
__global__ void __launch_bounds__(256) act_bwd_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ pre,
                                                      int64_t n8, bf16* __restrict__ dx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float g[8], z[8];
    load8(dy + i * 8, g);
    load8(pre + i * 8, z);
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] *= act_bwd(ACT, z[j]);
    store8(dx + i * 8, g);
  }
}

static int elementwise_grid(int64_t n8) {
  const int64_t want = (n8 + 255) / 256;
  const int64_t cap = (int64_t)row_sms() * 8;
  return (int)(want < cap ? want : cap);
}

extern "C" int smpk_bias_act_fwd(const void* x, const void* bias, int M, int N, int act, void* pre_out, void* y,
                                 void* stream) {
  SMPK_REQUIRE(x && bias && pre_out && y && M > 0 && N > 0 && N % 8 == 0, SMPK_ERR_BAD_ARG,
               "smpk_bias_act_fwd: bad arguments (N must be a multiple of 8)");
  const int64_t n8 = (int64_t)M * N / 8;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bf16 *xb = reinterpret_cast<const bf16*>(x), *bb = reinterpret_cast<const bf16*>(bias);
  bf16 *pb = reinterpret_cast<bf16*>(pre_out), *yb = reinterpret_cast<bf16*>(y);
  const int grid = elementwise_grid(n8);
  switch (act) {
    case SMPK_ACT_GELU_ERF: bias_act_fwd_kernel<SMPK_ACT_GELU_ERF><<<grid, 256, 0, st>>>(xb, bb, n8, N, pb, yb); break;
    case SMPK_ACT_GELU_TANH: bias_act_fwd_kernel<SMPK_ACT_GELU_TANH><<<grid, 256, 0, st>>>(xb, bb, n8, N, pb, yb); break;
    case SMPK_ACT_RELU: bias_act_fwd_kernel<SMPK_ACT_RELU><<<grid, 256, 0, st>>>(xb, bb, n8, N, pb, yb); break;
    default: SMPK_REQUIRE(false, SMPK_ERR_BAD_ARG, "smpk_bias_act_fwd: unknown activation %d", act);
  }
  return check_launch("smpk_bias_act_fwd");
}

extern "C" int smpk_act_bwd(const void* dy, const void* pre, int M, int N, int act, void* dx, void* stream) {
  SMPK_REQUIRE(dy && pre && dx && M > 0 && N > 0 && N % 8 == 0, SMPK_ERR_BAD_ARG,
               "smpk_act_bwd: bad arguments (N must be a multiple of 8)");
  const int64_t n8 = (int64_t)M * N / 8;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bf16 *gb = reinterpret_cast<const bf16*>(dy), *zb = reinterpret_cast<const bf16*>(pre);
  bf16* db = reinterpret_cast<bf16*>(dx);
  const int grid = elementwise_grid(n8);
  switch (act) {
    case SMPK_ACT_GELU_ERF: act_bwd_kernel<SMPK_ACT_GELU_ERF><<<grid, 256, 0, st>>>(gb, zb, n8, db); break;
    case SMPK_ACT_GELU_TANH: act_bwd_kernel<SMPK_ACT_GELU_TANH><<<grid, 256, 0, st>>>(gb, zb, n8, db); break;
    case SMPK_ACT_RELU: act_bwd_kernel<SMPK_ACT_RELU><<<grid, 256, 0, st>>>(gb, zb, n8, db); break;
    default: SMPK_REQUIRE(false, SMPK_ERR_BAD_ARG, "smpk_act_bwd: unknown activation %d", act);
  }
  return check_launch("smpk_act_bwd");
}

// Vectorised column partials: thread = 8 consecutive columns (one 16-B load per row),
// 8 row groups per block interleaved over a RPC-row chunk, summed in order in smem.
template <int RPC>
__global__ void __launch_bounds__(256) colsum_partial_vec_kernel(const bf16* x, int M, int N, int64_t ldx,
                                                                 float* partials) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sm[8][32 * 8 + 1];
  const int t = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int col0 = (blockIdx.x * 32 + t) * 8;
  const int r0 = blockIdx.y * RPC;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (col0 < N) {
    // all RPC/8 loads of this thread in flight at once
    uint4 u[RPC / 8];
#pragma unroll
    for (int k = 0; k < RPC / 8; ++k) {
      const int r = min(r0 + grp + 8 * k, M - 1);  // clamped (re-read) rows are masked below
      u[k] = *reinterpret_cast<const uint4*>(x + (int64_t)r * ldx + col0);
    }
#pragma unroll
    for (int k = 0; k < RPC / 8; ++k) {
      if (r0 + grp + 8 * k >= M) continue;
      const uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16x2(w[j]);
        acc[2 * j] += f.x;
        acc[2 * j + 1] += f.y;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) sm[grp][t * 8 + j] = acc[j];
  __syncthreads();
  const int c = threadIdx.x;  // 256 columns of this block
  const int col = blockIdx.x * 256 + c;
  if (col < N) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += sm[i][c];
    partials[(int64_t)blockIdx.y * N + col] = s;
  }
}

// rows per partial chunk: enough blocks to cover every SM twice, at most 128 rows (the 256-row
// variant holds 32 loads per thread in 202 registers: one block per SM, 2.2 TB/s at GPT-1.3B)
static int colsum_rpc(int M, int N) {
  const int cblocks = (N + 255) / 256;
  for (int rpc = 128; rpc > 64; rpc >>= 1)
    if ((int64_t)cblocks * ((M + rpc - 1) / rpc) >= 2 * row_sms()) return rpc;
  return 64;
}

extern "C" int64_t smpk_colsum_workspace(int M, int N) {
  if (M <= 0 || N <= 0) return 0;
  const int rpc = colsum_rpc(M, N);
  return (int64_t)((M + rpc - 1) / rpc) * N * 4;
}

extern "C" int smpk_colsum(const void* x, int M, int N, int64_t ldx, void* out, int out_f32, int accumulate,
                           void* workspace, int64_t workspace_bytes, void* stream) {
  SMPK_REQUIRE(M > 0 && N > 0 && x && out, SMPK_ERR_BAD_ARG, "smpk_colsum: bad arguments");
  const bool vec = (N % 8 == 0) && (ldx % 8 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
  const int rpc = vec ? colsum_rpc(M, N) : 256;
  const int chunks = (M + rpc - 1) / rpc;
  SMPK_REQUIRE(workspace && workspace_bytes >= (int64_t)chunks * N * 4, SMPK_ERR_BAD_ARG,
               "smpk_colsum: workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  dim3 g1((N + 255) / 256, chunks);
  float* ws = reinterpret_cast<float*>(workspace);
  const bf16* xb = reinterpret_cast<const bf16*>(x);
  if (vec) {
    if (rpc == 256) launch_pdl(colsum_partial_vec_kernel<256>, g1, 256, 0, st, xb, M, N, ldx, ws);
    else if (rpc == 128) launch_pdl(colsum_partial_vec_kernel<128>, g1, 256, 0, st, xb, M, N, ldx, ws);
    else launch_pdl(colsum_partial_vec_kernel<64>, g1, 256, 0, st, xb, M, N, ldx, ws);
  } else {
    launch_pdl(colsum_partial_kernel, g1, 256, 0, st, xb, M, N, ldx, 256, ws);
  }
  int rc = check_launch("smpk_colsum");
  if (rc) return rc;
  dim3 g2((N + 31) / 32, 1);
  colsum_reduce_launch(g2, ws, chunks, 1, N, out, nullptr, nullptr, out_f32, accumulate, st);
  return check_launch("smpk_colsum(reduce)");
}

#define SMPK_NV_CASE(NV_, KERNEL, CFG, ARGS) \
  case NV_:                                  \
    KERNEL<NV_><<<SMPK_UNPACK CFG>>> ARGS;   \
    break;
#define SMPK_DISPATCH_NV(NV_, KERNEL, CFG, ARGS)                                                 \
  switch (NV_) {                                                                                 \
    SMPK_NV_CASE(1, KERNEL, CFG, ARGS) SMPK_NV_CASE(2, KERNEL, CFG, ARGS)                        \
    SMPK_NV_CASE(4, KERNEL, CFG, ARGS) SMPK_NV_CASE(8, KERNEL, CFG, ARGS)                        \
    SMPK_NV_CASE(16, KERNEL, CFG, ARGS)                                                          \
    default:                                                                                     \
      set_last_error("unsupported key length");                                                 \
      return SMPK_ERR_UNSUPPORTED;                                                               \
  }

extern "C" int smpk_softmax_fwd(const void* scores, void* probs, void* probs_drop, const float* mask_add, int B,
                                int nh, int sq, int sk, float scale, int causal, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer,
                                int64_t sample_offset, int head_offset, int nh_global, void* stream) {
  const int nv = softmax_nv(sk);
  SMPK_REQUIRE(nv > 0 && sk % 8 == 0 && B > 0 && nh > 0 && sq > 0, SMPK_ERR_UNSUPPORTED,
               "smpk_softmax_fwd: key length %d unsupported (multiple of 8, <= 4096)", sk);
  SMPK_REQUIRE(scores && probs && (p_drop == 0.f || probs_drop), SMPK_ERR_BAD_ARG, "smpk_softmax_fwd: null argument");
  SMPK_REQUIRE(!causal || sq <= sk, SMPK_ERR_BAD_SHAPE, "smpk_softmax_fwd: causal needs sq <= sk");
  SoftmaxArgs a{reinterpret_cast<const bf16*>(scores), nullptr, reinterpret_cast<bf16*>(probs),
                reinterpret_cast<bf16*>(probs_drop), mask_add, B, nh, sq, sk, scale, p_drop, causal, seed,
                (uint32_t)layer, sample_offset, head_offset, nh_global};
  a.rng_step = rng_step;
  const int64_t rows = (int64_t)B * nh * sq;
  int64_t grid = (rows + 7) / 8;
  if (grid > row_sms() * 8) grid = row_sms() * 8;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  SMPK_DISPATCH_NV(nv, softmax_fwd_kernel, ((int)grid, ROW_THREADS, 0, st), (a));
  return check_launch("smpk_softmax_fwd");
}

extern "C" int smpk_softmax_bwd(const void* probs, const void* dprobs_drop, void* dscores, int B, int nh, int sq,
                                int sk, float scale, float p_drop, uint64_t seed, const uint64_t* rng_step, int layer, int64_t sample_offset,
                                int head_offset, int nh_global, void* stream) {
  const int nv = softmax_nv(sk);
  SMPK_REQUIRE(nv > 0 && sk % 8 == 0, SMPK_ERR_UNSUPPORTED, "smpk_softmax_bwd: key length %d unsupported", sk);
  SMPK_REQUIRE(probs && dprobs_drop && dscores, SMPK_ERR_BAD_ARG, "smpk_softmax_bwd: null argument");
  SoftmaxArgs a{reinterpret_cast<const bf16*>(probs), reinterpret_cast<const bf16*>(dprobs_drop),
                reinterpret_cast<bf16*>(dscores), nullptr, nullptr, B, nh, sq, sk, scale, p_drop, 0, seed,
                (uint32_t)layer, sample_offset, head_offset, nh_global};
  a.rng_step = rng_step;
  const int64_t rows = (int64_t)B * nh * sq;
  int64_t grid = (rows + 7) / 8;
  if (grid > row_sms() * 8) grid = row_sms() * 8;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  SMPK_DISPATCH_NV(nv, softmax_bwd_kernel, ((int)grid, ROW_THREADS, 0, st), (a));
  return check_launch("smpk_softmax_bwd");
}

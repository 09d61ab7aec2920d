// embed_ce.cu — embedding lookup / deterministic scatter-add and vocab-parallel
// softmax cross-entropy (sm_100a).
//
//   smpk_embed_fwd : out[t] = table[id_t - row_offset] if owned else 0  (+ pos_table[t % seq])
//                    (vocab-parallel: rank owns rows [row_offset, row_offset+rows_local);
//                     embedding-dim sharded: row_offset = 0, rows_local = V, table holds D/T columns)
//   smpk_embed_bwd : dtable[r] (+)= sum over tokens with id == row_offset + r of dY[t], summed in
//                    token order (owner-computes row blocks; no float atomics -> bit-deterministic)
//   smpk_vocab_ce_fwd_local : per row local max m_j, S_j = sum exp(l - m_j) over real columns,
//                    target logit if owned  -> stats [N, 3]
//   smpk_vocab_ce_combine   : combine T ranks' stats in rank order -> loss, global (m, S)
//   smpk_vocab_ce_bwd       : dlogits = (exp(l - m)/S - onehot) * g  on the local shard
//
// One warp per token row, 128-bit vector I/O, warp-shuffle max/sum reductions.
#include "smpk_common.cuh"

namespace smpk {

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------
// embedding forward
// ---------------------------------------------------------------------------
// thread per (token, 8-column vector): consecutive threads walk a row's 16-B vectors, then the
// next token -- coalesced for wide rows, and every lane busy for narrow ones (NCF: 8 columns per
// rank, one vector per token; a warp per token left 31 lanes idle)
__global__ void __launch_bounds__(256) embed_fwd_kernel(const int64_t* __restrict__ ids, int64_t n,
                                                        const bf16* __restrict__ table, int64_t ld_table,
                                                        int64_t row_offset, int64_t rows_local, int64_t vocab,
                                                        int dim, bf16* __restrict__ out, int64_t ld_out,
                                                        const bf16* __restrict__ pos_table, int64_t ld_pos, int seq,
                                                        unsigned long long* err_pos) {
  const bool vec = (dim % 8 == 0) && (ld_table % 8 == 0) && (ld_out % 8 == 0) && (ld_pos % 8 == 0);
  const int nvec = vec ? dim / 8 : dim;  // vectors (or scalars) per row
  const int64_t total = n * nvec;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx / nvec;
    const int c = (int)(idx - t * nvec);
    const int64_t id = __ldg(ids + t);
    if ((id < 0 || id >= vocab) && c == 0 && err_pos) atomicMin(err_pos, (unsigned long long)t);
    const int64_t loc = id - row_offset;
    const bool own = (id >= 0 && id < vocab) && loc >= 0 && loc < rows_local;
    const bf16* src = table + (own ? loc : 0) * ld_table;
    const bf16* ps = pos_table ? pos_table + (t % seq) * ld_pos : nullptr;
    bf16* dst = out + t * ld_out;
    if (vec) {
      uint4 u = own ? __ldg(reinterpret_cast<const uint4*>(src) + c) : make_uint4(0, 0, 0, 0);
      if (ps) {
        uint4 p = __ldg(reinterpret_cast<const uint4*>(ps) + c);
        uint32_t a[4] = {u.x, u.y, u.z, u.w}, b[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 fa = unpack_bf16x2(a[j]), fb = unpack_bf16x2(b[j]);
          a[j] = pack_bf16x2(fa.x + fb.x, fa.y + fb.y);
        }
        u = make_uint4(a[0], a[1], a[2], a[3]);
      }
      reinterpret_cast<uint4*>(dst)[c] = u;
    } else {
      float v = own ? bf2f(src[c]) : 0.f;
      if (ps) v += bf2f(ps[c]);
      dst[c] = f2bf(v);
    }
  }
}

// ---------------------------------------------------------------------------
// embedding backward: owner-computes over blocks of EB_ROWS local rows.
// Each CTA scans the token ids in order, compacts the positions that fall in its
// row block into shared memory (order preserved), then accumulates dY rows into
// fp32 registers in token order: bit-deterministic with no atomics.
// ---------------------------------------------------------------------------
constexpr int EB_ROWS = 8;
constexpr int EB_THREADS = 256;
constexpr int EB_LIST = 2048;  // matched-token capacity per scan batch

__global__ void __launch_bounds__(EB_THREADS) embed_bwd_kernel(const int64_t* __restrict__ ids, int64_t n,
                                                               const bf16* __restrict__ dy, int64_t ld_dy,
                                                               int64_t row_offset, int64_t rows_local, int dim,
                                                               void* dtable, int64_t ld_dt, int out_f32,
                                                               int accumulate, int64_t padding_row) {
  __shared__ int64_t list[EB_LIST];
  __shared__ int cnt;
  __shared__ int warp_counts[EB_THREADS / 32];
  const int64_t r0 = (int64_t)blockIdx.x * EB_ROWS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // each thread owns columns c = (tid + k*EB_THREADS) for k in [0, ceil(dim/EB_THREADS))
  constexpr int MAXK = 20;  // dim <= 5120
  float acc[EB_ROWS][MAXK];
#pragma unroll
  for (int r = 0; r < EB_ROWS; ++r)
#pragma unroll
    for (int k = 0; k < MAXK; ++k) acc[r][k] = 0.f;
  const int kmax = (dim + EB_THREADS - 1) / EB_THREADS;

  for (int64_t base = 0; base < n;) {
    if (tid == 0) cnt = 0;
    __syncthreads();
    // scan ids in chunks of EB_THREADS, compact in order until the list would overflow
    int64_t next = base;
    while (next < n) {
      const int64_t t = next + tid;
      bool hit = false;
      if (t < n) {
        const int64_t loc = ids[t] - row_offset - r0;
        hit = loc >= 0 && loc < EB_ROWS && (r0 + loc) < rows_local && (ids[t] != padding_row);
      }
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) warp_counts[warp] = __popc(m);
      __syncthreads();
      int before = 0, total = 0;
      for (int w = 0; w < EB_THREADS / 32; ++w) {
        if (w < warp) before += warp_counts[w];
        total += warp_counts[w];
      }
      const int cur = cnt;
      if (cur + total > EB_LIST) {  // uniform: process what we have first
        __syncthreads();
        break;
      }
      if (hit) list[cur + before + __popc(m & ((1u << lane) - 1))] = t;
      __syncthreads();
      if (tid == 0) cnt = cur + total;
      next += EB_THREADS;
      __syncthreads();
    }
    const int L = cnt;
    for (int i = 0; i < L; ++i) {
      const int64_t t = list[i];
      const int r = (int)(ids[t] - row_offset - r0);
      const bf16* src = dy + t * ld_dy;
#pragma unroll
      for (int k = 0; k < MAXK; ++k) {
        const int c = tid + k * EB_THREADS;
        if (k < kmax && c < dim) {
          const float v = bf2f(src[c]);
#pragma unroll
          for (int rr = 0; rr < EB_ROWS; ++rr)
            if (rr == r) acc[rr][k] += v;
        }
      }
    }
    base = next;
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < EB_ROWS; ++r) {
    const int64_t row = r0 + r;
    if (row >= rows_local) break;
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      const int c = tid + k * EB_THREADS;
      if (k < kmax && c < dim) {
        if (out_f32) {
          float* d = reinterpret_cast<float*>(dtable) + row * ld_dt + c;
          *d = accumulate ? *d + acc[r][k] : acc[r][k];
        } else {
          bf16* d = reinterpret_cast<bf16*>(dtable) + row * ld_dt + c;
          *d = f2bf(accumulate ? bf2f(*d) + acc[r][k] : acc[r][k]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// vocab-parallel cross-entropy
// ---------------------------------------------------------------------------
// number of non-padding columns of a shard covering [col_offset, col_offset + v_local)
__device__ __forceinline__ int real_cols(int v_local, int64_t vocab, int64_t col_offset) {
  const int64_t r = vocab - col_offset;
  return r <= 0 ? 0 : (r < v_local ? (int)r : v_local);
}

// stats[row] = {m_j, S_j, target logit if owned else 0, owned flag}
__global__ void __launch_bounds__(256) ce_local_kernel(const bf16* __restrict__ logits, int64_t ld, int64_t N,
                                                       int v_local, int64_t col_offset, int64_t vocab,
                                                       const int64_t* __restrict__ targets, int64_t ignore_index,
                                                       float4* __restrict__ stats) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_real = real_cols(v_local, vocab, col_offset);
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < N; row += (int64_t)gridDim.x * 8) {
    const bf16* l = logits + row * ld;
    float m = -INFINITY, s = 0.f;
    const bool vec = (ld % 8 == 0);
    int c = lane * 8;
    if (vec) {
      for (; c + 8 <= n_real; c += 256) {
        uint4 u = *reinterpret_cast<const uint4*>(l + c);
        uint32_t w[4] = {u.x, u.y, u.z, u.w};
        float v[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 f = unpack_bf16x2(w[j]);
          v[2 * j] = f.x;
          v[2 * j + 1] = f.y;
        }
        float cm = v[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) cm = fmaxf(cm, v[j]);
        const float nm = fmaxf(m, cm);
        s = s * __expf(m - nm);
#pragma unroll
        for (int j = 0; j < 8; ++j) s += __expf(v[j] - nm);
        m = nm;
      }
    } else {
      c = 0;
    }
    // scalar tail (or whole row when unaligned)
    for (int cc = (vec ? (n_real / 8) * 8 : 0) + lane; cc < n_real; cc += 32) {
      const float v = bf2f(l[cc]);
      const float nm = fmaxf(m, v);
      s = s * __expf(m - nm) + __expf(v - nm);
      m = nm;
    }
    // warp combine
    float gm = warp_max_f(m);
    float gs = warp_sum_f(m == -INFINITY ? 0.f : s * __expf(m - gm));
    const int64_t tg = targets[row];
    const int64_t loc = tg - col_offset;
    const bool own = tg != ignore_index && loc >= 0 && loc < n_real;
    if (lane == 0) {
      const float tl = own ? bf2f(l[loc]) : 0.f;
      stats[row] = make_float4(gm, gs, tl, own ? 1.f : 0.f);
    }
  }
}

// stats_all [T][N] float4, combined in ascending rank order.
__global__ void ce_combine_kernel(const float4* __restrict__ stats_all, int T, int64_t N,
                                  const int64_t* __restrict__ targets, int64_t ignore_index, float* __restrict__ loss,
                                  float2* __restrict__ ms) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= N) return;
  float m = -INFINITY;
  for (int j = 0; j < T; ++j) m = fmaxf(m, stats_all[(int64_t)j * N + row].x);
  float S = 0.f, tl = 0.f;
  for (int j = 0; j < T; ++j) {
    const float4 st = stats_all[(int64_t)j * N + row];
    if (st.x != -INFINITY) S += st.y * __expf(st.x - m);
    tl += st.z;
  }
  const bool valid = targets[row] != ignore_index;
  loss[row] = valid ? (logf(S) + m - tl) : 0.f;
  ms[row] = make_float2(m, S);
}

__global__ void __launch_bounds__(256) ce_bwd_kernel(const bf16* __restrict__ logits, int64_t ld, int64_t N,
                                                     int v_local, int64_t col_offset, int64_t vocab,
                                                     const int64_t* __restrict__ targets, int64_t ignore_index,
                                                     const float2* __restrict__ ms, const float* __restrict__ gloss,
                                                     float gscale, bf16* __restrict__ dlogits, int64_t ld_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_real = real_cols(v_local, vocab, col_offset);
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < N; row += (int64_t)gridDim.x * 8) {
    const int64_t tg = targets[row];
    const bool valid = tg != ignore_index;
    const float g = valid ? (gloss ? gloss[row] : 1.f) * gscale : 0.f;
    const float2 st = ms[row];
    const float inv = 1.f / st.y;
    const int64_t loc = tg - col_offset;
    const bf16* l = logits + row * ld;
    bf16* d = dlogits + row * ld_out;
    const bool vec = (ld % 8 == 0) && (ld_out % 8 == 0) && (v_local % 8 == 0);
    if (vec) {
      for (int c = lane * 8; c < v_local; c += 256) {
        uint4 u = *reinterpret_cast<const uint4*>(l + c);
        uint32_t w[4] = {u.x, u.y, u.z, u.w};
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 f = unpack_bf16x2(w[j]);
          const int c0 = c + 2 * j;
          float p0 = c0 < n_real ? __expf(f.x - st.x) * inv : 0.f;
          float p1 = c0 + 1 < n_real ? __expf(f.y - st.x) * inv : 0.f;
          if (c0 == loc) p0 -= 1.f;
          if (c0 + 1 == loc) p1 -= 1.f;
          o[j] = pack_bf16x2(p0 * g, p1 * g);
        }
        *reinterpret_cast<uint4*>(d + c) = make_uint4(o[0], o[1], o[2], o[3]);
      }
    } else {
      for (int c = lane; c < v_local; c += 32) {
        float p = c < n_real ? __expf(bf2f(l[c]) - st.x) * inv : 0.f;
        if (c == loc) p -= 1.f;
        d[c] = f2bf(p * g);
      }
    }
  }
}

}  // namespace smpk

using namespace smpk;

extern "C" int smpk_embed_fwd(const int64_t* ids, int64_t n, const void* table, int64_t ld_table, int64_t row_offset,
                              int64_t rows_local, int64_t vocab, int dim, void* out, int64_t ld_out,
                              const void* pos_table, int64_t ld_pos, int seq, unsigned long long* err_pos,
                              void* stream) {
  SMPK_REQUIRE(ids && table && out && dim > 0 && n >= 0, SMPK_ERR_BAD_ARG, "smpk_embed_fwd: bad arguments");
  SMPK_REQUIRE(!pos_table || seq > 0, SMPK_ERR_BAD_ARG, "smpk_embed_fwd: pos_table needs seq > 0");
  if (n == 0) return SMPK_OK;
  const int64_t work = n * (dim % 8 == 0 ? dim / 8 : dim);
  int64_t grid = (work + 255) / 256;
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  embed_fwd_kernel<<<(int)grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      ids, n, reinterpret_cast<const bf16*>(table), ld_table, row_offset, rows_local, vocab, dim,
      reinterpret_cast<bf16*>(out), ld_out, reinterpret_cast<const bf16*>(pos_table), ld_pos, seq, err_pos);
  return check_launch("smpk_embed_fwd");
}

extern "C" int smpk_embed_bwd(const int64_t* ids, int64_t n, const void* dy, int64_t ld_dy, int64_t row_offset,
                              int64_t rows_local, int dim, void* dtable, int64_t ld_dt, int out_f32, int accumulate,
                              int64_t padding_row, void* stream) {
  SMPK_REQUIRE(ids && dy && dtable && rows_local > 0, SMPK_ERR_BAD_ARG, "smpk_embed_bwd: bad arguments");
  SMPK_REQUIRE(dim > 0 && dim <= 20 * EB_THREADS, SMPK_ERR_UNSUPPORTED, "smpk_embed_bwd: dim %d > 5120", dim);
  const int64_t grid = (rows_local + EB_ROWS - 1) / EB_ROWS;
  embed_bwd_kernel<<<(unsigned)grid, EB_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      ids, n, reinterpret_cast<const bf16*>(dy), ld_dy, row_offset, rows_local, dim, dtable, ld_dt, out_f32,
      accumulate, padding_row);
  return check_launch("smpk_embed_bwd");
}

extern "C" int smpk_vocab_ce_fwd_local(const void* logits, int64_t ld, int64_t N, int v_local, int64_t col_offset,
                                       int64_t vocab, const int64_t* targets, int64_t ignore_index, float* stats,
                                       void* stream) {
  SMPK_REQUIRE(logits && targets && stats && v_local > 0, SMPK_ERR_BAD_ARG, "smpk_vocab_ce_fwd_local: bad args");
  if (N == 0) return SMPK_OK;
  int64_t grid = (N + 7) / 8;
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  ce_local_kernel<<<(int)grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const bf16*>(logits), ld, N, v_local, col_offset, vocab, targets, ignore_index,
      reinterpret_cast<float4*>(stats));
  return check_launch("smpk_vocab_ce_fwd_local");
}

extern "C" int smpk_vocab_ce_combine(const float* stats_all, int T, int64_t N, const int64_t* targets,
                                     int64_t ignore_index, float* loss, float* ms, void* stream) {
  SMPK_REQUIRE(stats_all && targets && loss && ms && T > 0, SMPK_ERR_BAD_ARG, "smpk_vocab_ce_combine: bad args");
  if (N == 0) return SMPK_OK;
  ce_combine_kernel<<<(unsigned)((N + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4*>(stats_all), T, N, targets, ignore_index, loss, reinterpret_cast<float2*>(ms));
  return check_launch("smpk_vocab_ce_combine");
}

extern "C" int smpk_vocab_ce_bwd(const void* logits, int64_t ld, int64_t N, int v_local, int64_t col_offset,
                                 int64_t vocab, const int64_t* targets, int64_t ignore_index, const float* ms,
                                 const float* grad_loss, float grad_scale, void* dlogits, int64_t ld_out,
                                 void* stream) {
  SMPK_REQUIRE(logits && targets && ms && dlogits, SMPK_ERR_BAD_ARG, "smpk_vocab_ce_bwd: bad args");
  if (N == 0) return SMPK_OK;
  int64_t grid = (N + 7) / 8;
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  ce_bwd_kernel<<<(int)grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const bf16*>(logits), ld, N, v_local, col_offset, vocab, targets, ignore_index,
      reinterpret_cast<const float2*>(ms), grad_loss, grad_scale, reinterpret_cast<bf16*>(dlogits), ld_out);
  return check_launch("smpk_vocab_ce_bwd");
}

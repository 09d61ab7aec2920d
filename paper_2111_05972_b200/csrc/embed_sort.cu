// embed_sort.cu — deterministic sort-based embedding backward (sm_100a).
//
//   dtable[r] (+)= sum of dy[t] over tokens t with ids[t] == row_offset + r
//
// for tables far larger than the batch (NCF: 10^8 rows per rank; SPEC.md:440-448,
// PAPER.md:424-426), where scanning the token list once per row block (smpk_embed_bwd) is
// O(rows * n).  Here the work is O(n log rows) and touches only the rows that occur:
//   1. keys: local row of every token (or a sentinel for tokens of other ranks / padding)
//   2. LSD radix sort of (key, token position), 8-bit digits, stable: equal rows keep token
//      order; every pass = per-tile digit histogram -> tile-ordered exclusive scan -> scatter
//      with an in-tile stable rank (warp __match_any + per-warp digit counters)
//   3. segmented sums over the sorted positions in fixed-size windows (lanes = tokens for narrow
//      rows, lanes = columns for wide rows) in a fixed order; runs that stay inside a window are
//      added to their table row directly (one fp32 read-modify-write per unique row); runs that
//      cross a window boundary leave per-window partials that one owner sums in window order.
// No float atomics anywhere: the result is bit-identical run to run.
#include <cstring>

#include "smpk_common.cuh"

namespace smpk {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 8;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 2048 keys per tile
constexpr int SEG_W_LARGE = 64;                  // window of the wide-row segmented sum

__global__ void __launch_bounds__(256) embed_keys_kernel(const int64_t* __restrict__ ids, int64_t n,
                                                         int64_t row_offset, int64_t rows_local, int64_t padding_row,
                                                         uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                         int* __restrict__ n_valid) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = false;
  if (t < n) {
    const int64_t id = ids[t];
    const int64_t loc = id - row_offset;
    valid = loc >= 0 && loc < rows_local && id != padding_row;
    keys[t] = valid ? (uint32_t)loc : (uint32_t)rows_local;  // sentinel sorts last
    vals[t] = (uint32_t)t;
  }
  const int c = __syncthreads_count(valid);  // one atomic per block (per-warp atomics on one word serialised)
  if (threadIdx.x == 0 && c) atomicAdd(n_valid, c);
}

// digits of BITS bits (8 or 9: the row count of the table decides how many passes the keys need;
// 27-bit keys of a 1e8-row table take three 9-bit passes instead of four 8-bit ones)
template <int BITS>
__global__ void __launch_bounds__(RS_THREADS) radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t n,
                                                                int shift, int num_tiles, int* __restrict__ counts) {
  constexpr int BINS = 1 << BITS;
  __shared__ int hist[BINS];
  for (int d = threadIdx.x; d < BINS; d += RS_THREADS) hist[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll
  for (int k = 0; k < RS_ITEMS; ++k) {
    const int64_t i = base + k * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&hist[(keys[i] >> shift) & (BINS - 1)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < BINS; d += RS_THREADS) counts[(int64_t)d * num_tiles + blockIdx.x] = hist[d];
}

// counts[d][tile] -> exclusive prefix over the tiles of digit d (block d, coalesced 1024-wide chunks
// with a carried block scan) and digit_tot[d]; radix_digit_kernel turns the totals into the digit
// bases.  Global position of (digit d, tile t) = digit_base[d] + counts[d][t].
constexpr int SCAN_THREADS = 256;
__global__ void __launch_bounds__(SCAN_THREADS) radix_scan_kernel(int* __restrict__ counts, int num_tiles,
                                                                  int* __restrict__ digit_tot) {
  // 1024-entry chunks: 4 consecutive tiles per thread, warp shuffle scan, 8 warp totals in smem
  __shared__ int wsum[SCAN_THREADS / 32];
  int* row = counts + (int64_t)blockIdx.x * num_tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int carry = 0;
  for (int base = 0; base < num_tiles; base += 4 * SCAN_THREADS) {
    const int t0 = base + threadIdx.x * 4;
    int v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = t0 + k < num_tiles ? row[t0 + k] : 0;
    const int sum = (v[0] + v[1]) + (v[2] + v[3]);
    int x = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = lane < SCAN_THREADS / 32 ? wsum[lane] : 0;
#pragma unroll
      for (int off = 1; off < SCAN_THREADS / 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += y;
      }
      if (lane < SCAN_THREADS / 32) wsum[lane] = w;
    }
    __syncthreads();
    int e = carry + (warp > 0 ? wsum[warp - 1] : 0) + x - sum;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (t0 + k < num_tiles) {
        row[t0 + k] = e;
        e += v[k];
      }
    carry += wsum[SCAN_THREADS / 32 - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) digit_tot[blockIdx.x] = carry;
}

template <int BITS>
__global__ void __launch_bounds__(1 << BITS) radix_digit_kernel(int* __restrict__ digit_tot) {
  constexpr int BINS = 1 << BITS;
  __shared__ int part[BINS];
  const int d = threadIdx.x;
  const int v = digit_tot[d];
  part[d] = v;
  __syncthreads();
  for (int off = 1; off < BINS; off <<= 1) {
    const int o = d >= off ? part[d - off] : 0;
    __syncthreads();
    part[d] += o;
    __syncthreads();
  }
  digit_tot[d] = part[d] - v;  // exclusive: the digit's base
}

// Stable scatter: warp w of a tile owns the tile's elements [w*256, w*256+256) in order; each
// iteration ranks 32 consecutive elements with __match_any_sync against per-warp digit counters.
template <int BITS>
__global__ void __launch_bounds__(RS_THREADS) radix_scatter_kernel(const uint32_t* __restrict__ keys_in,
                                                                   const uint32_t* __restrict__ vals_in, int64_t n,
                                                                   int shift, int num_tiles,
                                                                   const int* __restrict__ counts,
                                                                   const int* __restrict__ digit_base,
                                                                   uint32_t* __restrict__ keys_out,
                                                                   uint32_t* __restrict__ vals_out) {
  constexpr int BINS = 1 << BITS;
  __shared__ int wc[RS_THREADS / 32][BINS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int d = lane; d < BINS; d += 32) wc[warp][d] = 0;
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE + warp * 256;
  uint32_t key[RS_ITEMS], val[RS_ITEMS];
  int rank[RS_ITEMS];
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    const int64_t i = base + it * 32 + lane;
    const bool ok = i < n;
    key[it] = ok ? keys_in[i] : 0u;
    val[it] = ok ? vals_in[i] : 0u;
    const int d = ok ? (int)((key[it] >> shift) & (BINS - 1)) : BINS + lane;  // out-of-range lanes match nobody
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int before = __popc(peers & ((1u << lane) - 1));
    int cnt = 0;
    if (ok) cnt = wc[warp][d];
    rank[it] = cnt + before;
    __syncwarp();
    if (ok && before == 0) wc[warp][d] = cnt + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix of the per-warp counters, per digit, in warp order
  for (int d = threadIdx.x; d < BINS; d += RS_THREADS) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < RS_THREADS / 32; ++w) {
      const int v = wc[w][d];
      wc[w][d] = s;
      s += v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < RS_ITEMS; ++it) {
    const int64_t i = base + it * 32 + lane;
    if (i < n) {
      const int d = (int)((key[it] >> shift) & (BINS - 1));
      const int64_t pos = (int64_t)digit_base[d] + counts[(int64_t)d * num_tiles + blockIdx.x] + wc[warp][d] + rank[it];
      keys_out[pos] = key[it];
      vals_out[pos] = val[it];
    }
  }
}

struct SegArgs {
  const uint32_t* keys;  // sorted local rows (valid prefix [0, n_valid))
  const uint32_t* vals;  // token positions
  const int* n_valid;
  const bf16* dy;
  int64_t ld_dy;
  int dim;
  void* dtable;
  int64_t ld_dt;
  int out_f32;
  int window;
  float* partial;  // [num_windows][2][dim]: head (continuation) and tail (open run started here)
};

__device__ __forceinline__ void rmw_row8(const SegArgs& a, uint32_t row, int c0, const float (&v)[8]) {
  if (a.out_f32) {
    float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.dtable) + (int64_t)row * a.ld_dt + c0);
    float4 x0 = d[0], x1 = d[1];
    x0.x += v[0]; x0.y += v[1]; x0.z += v[2]; x0.w += v[3];
    x1.x += v[4]; x1.y += v[5]; x1.z += v[6]; x1.w += v[7];
    d[0] = x0;
    d[1] = x1;
  } else {
    uint4* d = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(a.dtable) + (int64_t)row * a.ld_dt + c0);
    uint4 u = *d;
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16x2(w[j]);
      w[j] = pack_bf16x2(f.x + v[2 * j], f.y + v[2 * j + 1]);
    }
    *d = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__device__ __forceinline__ void load_dy8(const SegArgs& a, uint32_t pos, int c0, float (&v)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(a.dy + (int64_t)pos * a.ld_dy + c0);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = unpack_bf16x2(w[j]);
    v[2 * j] = f.x;
    v[2 * j + 1] = f.y;
  }
}

// Narrow rows (dim <= 64): warp per window of 32 sorted tokens, lane = token, NV 8-column vectors
// per lane; a fixed Hillis-Steele segmented scan across lanes sums each run.
template <int NV>
__global__ void __launch_bounds__(256) seg_small_kernel(const SegArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // window
  const int nv = *a.n_valid;
  const int64_t i0 = w * 32;
  if (i0 >= nv) return;
  const int64_t i = i0 + lane;
  const bool in = i < nv;
  const uint32_t key = in ? a.keys[i] : 0xffffffffu;
  float v[NV][8];
#pragma unroll
  for (int c = 0; c < NV; ++c) {
    if (in && c * 8 < a.dim) {
      load_dy8(a, a.vals[i], c * 8, v[c]);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[c][e] = 0.f;
    }
  }
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const uint32_t kprev = __shfl_up_sync(0xffffffffu, key, s);
#pragma unroll
    for (int c = 0; c < NV; ++c)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float o = __shfl_up_sync(0xffffffffu, v[c][e], s);
        if (lane >= s && kprev == key) v[c][e] += o;
      }
  }
  const uint32_t knext = __shfl_down_sync(0xffffffffu, key, 1);
  if (!in) return;
  const bool last_in_win = (lane == 31) || (i + 1 >= nv);
  const bool run_end_here = last_in_win ? (i + 1 >= nv || a.keys[i + 1] != key) : (knext != key);
  if (!(run_end_here || last_in_win)) return;  // only each run's last lane in the window writes
  // the run's first element in the window is lane 0 if keys[i0] == key; it started in an
  // earlier window iff that element continues the previous window's last key
  const uint32_t k0 = a.keys[i0];
  const bool starts_in_window = !(k0 == key && i0 > 0 && a.keys[i0 - 1] == key);
  const int dim = a.dim;
  float* head = a.partial + (w * 2 + 0) * (int64_t)dim;
  float* tail = a.partial + (w * 2 + 1) * (int64_t)dim;
  if (starts_in_window && run_end_here) {
#pragma unroll
    for (int c = 0; c < NV; ++c)
      if (c * 8 < dim) rmw_row8(a, key, c * 8, v[c]);
  } else if (!starts_in_window) {  // continuation of an earlier window's run (maybe still open)
#pragma unroll
    for (int c = 0; c < NV; ++c)
      if (c * 8 < dim)
#pragma unroll
        for (int e = 0; e < 8; ++e) head[c * 8 + e] = v[c][e];
  } else {  // open run starting here, continuing into the next window
#pragma unroll
    for (int c = 0; c < NV; ++c)
      if (c * 8 < dim)
#pragma unroll
        for (int e = 0; e < 8; ++e) tail[c * 8 + e] = v[c][e];
  }
}

// Wide rows (dim > 64): CTA per window of SEG_W_LARGE sorted tokens, thread = 8-column vector,
// tokens summed sequentially in sorted (= token) order.
__global__ void __launch_bounds__(256) seg_large_kernel(const SegArgs a) {
  const int nv = *a.n_valid;
  const int64_t w = blockIdx.x;
  const int64_t i0 = w * SEG_W_LARGE;
  if (i0 >= nv) return;
  const int64_t i1 = min((int64_t)nv, i0 + SEG_W_LARGE);
  const int dim = a.dim;
  float* head = a.partial + (w * 2 + 0) * (int64_t)dim;
  float* tail = a.partial + (w * 2 + 1) * (int64_t)dim;
  const bool first_cont = i0 > 0 && a.keys[i0 - 1] == a.keys[i0];
  for (int c0 = threadIdx.x * 8; c0 < dim; c0 += blockDim.x * 8) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    bool cont = first_cont;
    for (int64_t i = i0; i < i1; ++i) {
      const uint32_t key = a.keys[i];
      float v[8];
      load_dy8(a, a.vals[i], c0, v);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += v[e];
      const bool ends = (i + 1 >= nv) || a.keys[i + 1] != key;
      if (ends || i + 1 == i1) {
        float* dst = nullptr;
        if (cont) dst = head;            // continuation of an earlier window's run
        else if (!ends) dst = tail;       // open run starting here
        if (dst) {
#pragma unroll
          for (int e = 0; e < 8; ++e) dst[c0 + e] = acc[e];
        } else {
          rmw_row8(a, key, c0, acc);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        cont = false;
      }
    }
  }
}

// A run crossing windows is owned by the window where it starts (tail partial): it adds the head
// partials of the following windows up to the one where the run ends, then does one
// read-modify-write.  The window range is found by binary search on the sorted keys and summed in
// parallel with a fixed shape (window lanes stride the range in order, then a fixed tree), so a
// Zipf-hot row spanning hundreds of windows costs a few microseconds, deterministically.
__global__ void __launch_bounds__(256) seg_fixup_kernel(const SegArgs a, int num_windows) {
  __shared__ float red[256 * 8];
  const int64_t w = blockIdx.x;
  const int nv = *a.n_valid;
  const int W = a.window;
  const int64_t last = min((int64_t)nv, (w + 1) * W) - 1;
  if (w * W >= nv || last + 1 >= nv) return;
  const uint32_t key = a.keys[last];
  if (a.keys[last + 1] != key) return;  // no run leaves this window
  const int64_t i0 = w * W;
  if (a.keys[i0] == key && i0 > 0 && a.keys[i0 - 1] == key) return;  // an earlier window owns it
  // last index of the run: binary search in (last, nv)
  int64_t lo = last + 1, hi = nv - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (a.keys[mid] == key) lo = mid; else hi = mid - 1;
  }
  const int64_t u0 = w + 1, u1 = lo / W;  // windows holding head partials of this run
  const int64_t K = u1 - u0 + 1;
  const int dim = a.dim;
  const int nvec = dim / 8;
  int wl = 1;  // window lanes: a power of two with wl * nvec <= 256
  while (nvec < 256 && wl * 2 * nvec <= 256) wl *= 2;
  const int c = threadIdx.x % nvec, lane = threadIdx.x / nvec;
  for (int cv = c; cv < nvec; cv += (nvec >= 256 ? 256 : nvec)) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (lane < wl) {
      for (int64_t k = lane; k < K; k += wl) {
        const float* head = a.partial + ((u0 + k) * 2 + 0) * (int64_t)dim + cv * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += head[e];
      }
    }
    if (wl > 1) {  // fixed tree over the window lanes
      __syncthreads();
      if (lane < wl)
#pragma unroll
        for (int e = 0; e < 8; ++e) red[(lane * nvec + c) * 8 + e] = acc[e];
      __syncthreads();
      for (int s = wl >> 1; s > 0; s >>= 1) {
        if (lane < s)
#pragma unroll
          for (int e = 0; e < 8; ++e) red[(lane * nvec + c) * 8 + e] += red[((lane + s) * nvec + c) * 8 + e];
        __syncthreads();
      }
      if (lane != 0) continue;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = red[c * 8 + e];
    }
    const float* tail = a.partial + (w * 2 + 1) * (int64_t)dim + cv * 8;
    float tot[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) tot[e] = tail[e] + acc[e];
    rmw_row8(a, key, cv * 8, tot);
  }
}

static int bits_for(int64_t v) {
  int b = 0;
  while (b < 32 && (v >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

static int64_t align256(int64_t b) { return (b + 255) / 256 * 256; }

}  // namespace smpk

using namespace smpk;

static int64_t seg_windows(int64_t n, int dim) {
  const int W = dim <= 64 ? 32 : SEG_W_LARGE;
  return (n + W - 1) / W;
}

extern "C" int64_t smpk_embed_bwd_sorted_workspace(int64_t n, int64_t rows_local, int dim) {
  (void)rows_local;
  const int64_t tiles = (n + RS_TILE - 1) / RS_TILE;
  return align256(4 * n) * 4 + align256(512 * tiles * 4) + 2048 + 256 + align256(seg_windows(n, dim) * 2 * dim * 4);
}

extern "C" int smpk_embed_bwd_sorted(const int64_t* ids, int64_t n, const void* dy, int64_t ld_dy,
                                     int64_t row_offset, int64_t rows_local, int dim, void* dtable, int64_t ld_dt,
                                     int out_f32, int accumulate, int64_t padding_row, void* workspace,
                                     int64_t workspace_bytes, void* stream) {
  SMPK_REQUIRE(ids && dy && dtable && n >= 0 && rows_local > 0 && dim > 0, SMPK_ERR_BAD_ARG,
               "smpk_embed_bwd_sorted: bad arguments");
  SMPK_REQUIRE(rows_local < 0xffffffffLL && n < (1LL << 31), SMPK_ERR_UNSUPPORTED,
               "smpk_embed_bwd_sorted: rows_local / n too large");
  SMPK_REQUIRE(dim % 8 == 0 && ld_dy % 8 == 0 && ld_dt % 8 == 0 && dim <= 8192, SMPK_ERR_UNSUPPORTED,
               "smpk_embed_bwd_sorted: dim and leading dims must be multiples of 8 (<= 8192)");
  SMPK_REQUIRE(workspace_bytes >= smpk_embed_bwd_sorted_workspace(n, rows_local, dim), SMPK_ERR_BAD_ARG,
               "smpk_embed_bwd_sorted: workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t esz = out_f32 ? 4 : 2;
  if (!accumulate) {
    cudaError_t e = cudaMemset2DAsync(dtable, (size_t)ld_dt * esz, 0, (size_t)dim * esz, (size_t)rows_local, st);
    SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_embed_bwd_sorted: memset %s", cudaGetErrorString(e));
  }
  if (n == 0) return SMPK_OK;
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  const int64_t kb = align256(4 * n);
  uint32_t* k0 = reinterpret_cast<uint32_t*>(ws);
  uint32_t* v0 = reinterpret_cast<uint32_t*>(ws + kb);
  uint32_t* k1 = reinterpret_cast<uint32_t*>(ws + 2 * kb);
  uint32_t* v1 = reinterpret_cast<uint32_t*>(ws + 3 * kb);
  const int tiles = (int)((n + RS_TILE - 1) / RS_TILE);
  int* counts = reinterpret_cast<int*>(ws + 4 * kb);
  int* digit_base = reinterpret_cast<int*>(ws + 4 * kb + align256(512LL * tiles * 4));
  int* n_valid = reinterpret_cast<int*>(ws + 4 * kb + align256(512LL * tiles * 4) + 2048);
  float* partial = reinterpret_cast<float*>(ws + 4 * kb + align256(512LL * tiles * 4) + 2048 + 256);
  cudaMemsetAsync(n_valid, 0, sizeof(int), st);
  embed_keys_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ids, n, row_offset, rows_local, padding_row, k0, v0,
                                                                  n_valid);
  int rc = check_launch("smpk_embed_bwd_sorted(keys)");
  if (rc) return rc;
  const int nbits = bits_for(rows_local);  // keys in [0, rows_local] (sentinel included)
  const int bits = ((nbits + 7) / 8) * 9 >= nbits + 9 ? 9 : 8;  // 9-bit digits when they save a pass
  for (int shift = 0; shift < nbits; shift += bits) {
    if (bits == 9) {
      radix_hist_kernel<9><<<tiles, RS_THREADS, 0, st>>>(k0, n, shift, tiles, counts);
      radix_scan_kernel<<<512, SCAN_THREADS, 0, st>>>(counts, tiles, digit_base);
      radix_digit_kernel<9><<<1, 512, 0, st>>>(digit_base);
      radix_scatter_kernel<9><<<tiles, RS_THREADS, 0, st>>>(k0, v0, n, shift, tiles, counts, digit_base, k1, v1);
    } else {
      radix_hist_kernel<8><<<tiles, RS_THREADS, 0, st>>>(k0, n, shift, tiles, counts);
      radix_scan_kernel<<<256, SCAN_THREADS, 0, st>>>(counts, tiles, digit_base);
      radix_digit_kernel<8><<<1, 256, 0, st>>>(digit_base);
      radix_scatter_kernel<8><<<tiles, RS_THREADS, 0, st>>>(k0, v0, n, shift, tiles, counts, digit_base, k1, v1);
    }
    rc = check_launch("smpk_embed_bwd_sorted(radix)");
    if (rc) return rc;
    uint32_t* t = k0;
    k0 = k1;
    k1 = t;
    t = v0;
    v0 = v1;
    v1 = t;
  }
  SegArgs a{k0, v0, n_valid, reinterpret_cast<const bf16*>(dy), ld_dy, dim, dtable, ld_dt, out_f32, 0, partial};
  const int64_t nw = seg_windows(n, dim);
  if (dim <= 64) {
    a.window = 32;
    const unsigned grid = (unsigned)((nw * 32 + 255) / 256);
    switch ((dim + 7) / 8) {
      case 1: seg_small_kernel<1><<<grid, 256, 0, st>>>(a); break;
      case 2: seg_small_kernel<2><<<grid, 256, 0, st>>>(a); break;
      case 3:
      case 4: seg_small_kernel<4><<<grid, 256, 0, st>>>(a); break;
      default: seg_small_kernel<8><<<grid, 256, 0, st>>>(a); break;
    }
  } else {
    a.window = SEG_W_LARGE;
    seg_large_kernel<<<(unsigned)nw, 256, 0, st>>>(a);
  }
  rc = check_launch("smpk_embed_bwd_sorted(segments)");
  if (rc) return rc;
  seg_fixup_kernel<<<(unsigned)nw, 256, 0, st>>>(a, (int)nw);
  return check_launch("smpk_embed_bwd_sorted(fixup)");
}

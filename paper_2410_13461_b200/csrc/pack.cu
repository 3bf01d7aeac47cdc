// Weight-format kernels: device quantizer, bit-plane packer/unpacker,
// prefix-code reader, bit-exact dequantizer and the embedding row gather.
//
// Reference: pkg/src/pmpd/quant.py (quantize_tensor 157-191, BitPlaneStore
// 71-109, dequantize 199-215) and tinylm.py:334 (embedding gather).
#include <cuda_fp16.h>

#include "layout.cuh"
#include "pmpd_common.cuh"
#include "pmpd_internal.h"

namespace pmpd {

std::string& last_error_slot() {
  static thread_local std::string s;
  return s;
}

int num_sms() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || cached <= 0)
      cached = 148;
  }
  return cached;
}

namespace {

constexpr int kThreads = 256;

inline unsigned blocks_for(int64_t n, int per = kThreads) { return (unsigned)((n + per - 1) / per); }

// ------------------------------------------------------------------ quantizer
template <typename T>
__device__ __forceinline__ double load_w(const T* w, int64_t i);
template <>
__device__ __forceinline__ double load_w<float>(const float* w, int64_t i) {
  return (double)w[i];
}
template <>
__device__ __forceinline__ double load_w<double>(const double* w, int64_t i) {
  return w[i];
}
template <>
__device__ __forceinline__ double load_w<__half>(const __half* w, int64_t i) {
  return (double)__half2float(w[i]);
}

// One thread per (row, group): float64 min/max, f32 scales, codes against the
// f32-rounded scales with round-half-away (floor(x + 0.5)) and clamping —
// the exact IEEE operation sequence of quant.py:177-189.
template <typename T>
__global__ void quantize_kernel(const T* __restrict__ w, int rows, int cols, int gs, int groups, int levels,
                                uint8_t* __restrict__ codes, float* __restrict__ mins, float* __restrict__ deltas,
                                int* __restrict__ nonfinite) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)rows * groups) return;
  const int r = (int)(gid / groups), g = (int)(gid % groups);
  const int c0 = g * gs, c1 = min(cols, c0 + gs);
  const int64_t base = (int64_t)r * cols;
  double lo = 0.0, hi = 0.0;
  bool bad = false;
  for (int c = c0; c < c1; ++c) {
    const double v = load_w<T>(w, base + c);
    bad |= !isfinite(v);
    if (c == c0) {
      lo = v;
      hi = v;
    } else {
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
  }
  if (bad) atomicExch(nonfinite, 1);
  const float m32 = __double2float_rn(lo);
  const float d32 = __double2float_rn(__ddiv_rn(__dsub_rn(hi, lo), (double)levels));
  mins[gid] = m32;
  deltas[gid] = d32;
  const double md = (double)m32, dd = (double)d32;
  for (int c = c0; c < c1; ++c) {
    double q = 0.0;
    if (dd > 0.0) q = __ddiv_rn(__dsub_rn(load_w<T>(w, base + c), md), dd);
    q = floor(__dadd_rn(q, 0.5));
    q = fmin(fmax(q, 0.0), (double)levels);
    codes[base + c] = (uint8_t)q;
  }
}

// Reference plane bytes from codes: plane j = bit (p_max-1-j), flat row-major
// index i -> byte i>>3 bit i&7 (np.packbits bitorder="little", quant.py:89-93).
__global__ void planes_from_codes_kernel(const uint8_t* __restrict__ codes, int64_t n, int p_max, int64_t pbytes,
                                         uint8_t* __restrict__ planes) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= pbytes * p_max) return;
  const int j = (int)(id / pbytes);
  const int64_t byte = id % pbytes;
  const int bj = p_max - 1 - j;
  uint32_t out = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const int64_t i = byte * 8 + b;
    if (i < n) out |= ((codes[i] >> bj) & 1u) << b;
  }
  planes[id] = (uint8_t)out;
}

// ------------------------------------------------------------------ tiled pack
struct Geo {
  int rows, cols, gs, p_max, layout, n, k, nt, kt, groups;
  int64_t plane_bytes;
};

__host__ __device__ __forceinline__ void nk_to_ref(const Geo& g, int n, int k, int* r, int* c) {
  if (g.layout == PMPD_LAYOUT_KN) {
    *r = k;
    *c = n;
  } else {
    *r = n;
    *c = k;
  }
}

__device__ __forceinline__ uint32_t ref_bit(const uint8_t* planes, int64_t pbytes, int j, int64_t flat) {
  return (planes[(int64_t)j * pbytes + (flat >> 3)] >> (flat & 7)) & 1u;
}

// One thread per packed u32 word (plane j, tile, lane, word w).
__global__ void pack_planes_kernel(Geo g, const uint8_t* __restrict__ ref, int64_t ref_pbytes,
                                   uint32_t* __restrict__ out) {
  const int64_t words_per_plane = g.plane_bytes / 4;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= words_per_plane * g.p_max) return;
  const int j = (int)(id / words_per_plane);
  const int64_t wi = id % words_per_plane;
  const int64_t tile = wi / 128;
  const int lw = (int)(wi % 128), lane = lw >> 2, w = lw & 3;
  const int ng = (int)(tile / g.kt), kt = (int)(tile % g.kt);
  const int bj = g.p_max - 1 - j;
  uint32_t word = 0;
  for (int t = 0; t < 4; ++t)
    for (int s = 0; s < 8; ++s) {
      int nl, kl;
      tile_inverse(g.layout == PMPD_LAYOUT_KN, lane, w, t, s, &nl, &kl);
      const int n = ng * kTile + nl, k = kt * kTile + kl;
      if (n >= g.n || k >= g.k) continue;
      int r, c;
      nk_to_ref(g, n, k, &r, &c);
      word |= ref_bit(ref, ref_pbytes, j, (int64_t)r * g.cols + c) << tile_bitpos(t, s, bj);
    }
  out[id] = word;
}

// One thread per (tile, i in [0,128)): steps then mins.
__global__ void pack_scales_kernel(Geo g, const float* __restrict__ mins, const float* __restrict__ deltas,
                                   float* __restrict__ out) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ntiles = (int64_t)g.nt * g.kt;
  if (id >= ntiles * 128) return;
  const int64_t tile = id / 128;
  const int i = (int)(id % 128), which = i >> 6, q = i & 63;
  const int ng = (int)(tile / g.kt), kt = (int)(tile % g.kt);
  float v = 0.f;
  if (g.layout == PMPD_LAYOUT_KN) {
    const int k = kt * kTile + q, grp = ng * kTile / g.gs;
    if (k < g.k) v = (which ? mins : deltas)[(int64_t)k * g.groups + grp];
  } else {
    const int gq = q >> 3, t = (q & 7) >> 1, h = q & 1;
    const int n = ng * kTile + 16 * t + gq + 8 * h, grp = kt * kTile / g.gs;
    if (n < g.n) v = (which ? mins : deltas)[(int64_t)n * g.groups + grp];
  }
  out[id] = v;
}

// KN aux block: 1 / max_k step[k][group(n-tile)] per n-tile (0 if all steps are 0).
// The decode GEMV scales its integer activations by it so that the int16
// operand x*step*32767/(max|x| * max step) never overflows.
__global__ void pack_aux_kernel(Geo g, const float* __restrict__ deltas, float* __restrict__ aux) {
  const int ng = blockIdx.x;
  const int grp = ng * kTile / g.gs;
  float mx = 0.f;
  for (int k = threadIdx.x; k < g.k; k += blockDim.x) mx = fmaxf(mx, deltas[(int64_t)k * g.groups + grp]);
  mx = warp_max(mx);
  __shared__ float sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) mx = fmaxf(mx, sh[i]);
    aux[ng] = mx > 0.f ? 1.f / mx : 0.f;
  }
}

// code of reference element (r, c) read from the top p planes of any layout
__device__ __forceinline__ uint32_t load_code(const Geo& g, const uint8_t* base, int r, int c, int p) {
  uint32_t code = 0;
  if (g.layout == PMPD_LAYOUT_REF) {
    const int64_t flat = (int64_t)r * g.cols + c;
    for (int j = 0; j < p; ++j) code = (code << 1) | ref_bit(base, g.plane_bytes, j, flat);
    return code;
  }
  int n, k;
  if (g.layout == PMPD_LAYOUT_KN) {
    n = c;
    k = r;
  } else {
    n = r;
    k = c;
  }
  const int ng = n >> 6, kt = k >> 6;
  const TileCoord tc = tile_coord(g.layout == PMPD_LAYOUT_KN, n & 63, k & 63);
  const int64_t word = ((int64_t)ng * g.kt + kt) * 128 + tile_word(tc.lane, tc.w);
  const uint32_t* pl = reinterpret_cast<const uint32_t*>(base);
  for (int j = 0; j < p; ++j) {
    const uint32_t v = pl[(int64_t)j * (g.plane_bytes / 4) + word];
    code = (code << 1) | ((v >> tile_bitpos(tc.t, tc.s, g.p_max - 1 - j)) & 1u);
  }
  return code;
}

__device__ __forceinline__ void load_scale(const Geo& g, const uint8_t* base, int r, int c, float* mn, float* dl) {
  const uint8_t* sb = base + (int64_t)g.p_max * g.plane_bytes;
  const int grp = c / g.gs;
  if (g.layout == PMPD_LAYOUT_REF) {
    const float* m = reinterpret_cast<const float*>(sb);
    const int64_t off = (int64_t)g.rows * g.groups;
    *mn = m[(int64_t)r * g.groups + grp];
    *dl = m[off + (int64_t)r * g.groups + grp];
    return;
  }
  int n, k;
  if (g.layout == PMPD_LAYOUT_KN) {
    n = c;
    k = r;
  } else {
    n = r;
    k = c;
  }
  const int64_t tile = (int64_t)(n >> 6) * g.kt + (k >> 6);
  const float* blk = reinterpret_cast<const float*>(sb) + tile * 128;
  const int q = (g.layout == PMPD_LAYOUT_KN) ? (k & 63) : nk_scale_slot(n & 63);
  *dl = blk[q];
  *mn = blk[64 + q];
}

// bucket index of quant.py:212-215 as an exact f32 integer
__device__ __forceinline__ float bucket(uint32_t code, int p, int p_max) {
  if (p == p_max) return (float)code;
  const int m = p_max - p;
  return (float)((code << m) + (1u << (m - 1)));
}

__global__ void unpack_planes_kernel(Geo g, const uint8_t* __restrict__ base, int64_t ref_pbytes,
                                     uint8_t* __restrict__ ref) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= ref_pbytes * g.p_max) return;
  const int j = (int)(id / ref_pbytes);
  const int64_t byte = id % ref_pbytes;
  const int64_t n_el = (int64_t)g.rows * g.cols;
  const uint32_t* pl = reinterpret_cast<const uint32_t*>(base) + (int64_t)j * (g.plane_bytes / 4);
  uint32_t out = 0;
  for (int b = 0; b < 8; ++b) {
    const int64_t flat = byte * 8 + b;
    if (flat >= n_el) break;
    const int r = (int)(flat / g.cols), c = (int)(flat % g.cols);
    const int n = (g.layout == PMPD_LAYOUT_KN) ? c : r;
    const int k = (g.layout == PMPD_LAYOUT_KN) ? r : c;
    const TileCoord tc = tile_coord(g.layout == PMPD_LAYOUT_KN, n & 63, k & 63);
    const int64_t word = ((int64_t)(n >> 6) * g.kt + (k >> 6)) * 128 + tile_word(tc.lane, tc.w);
    out |= ((pl[word] >> tile_bitpos(tc.t, tc.s, g.p_max - 1 - j)) & 1u) << b;
  }
  ref[id] = (uint8_t)out;
}

__global__ void unpack_scales_kernel(Geo g, const uint8_t* __restrict__ base, float* __restrict__ mins,
                                     float* __restrict__ deltas) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)g.rows * g.groups) return;
  const int r = (int)(id / g.groups), grp = (int)(id % g.groups);
  float mn, dl;
  load_scale(g, base, r, grp * g.gs, &mn, &dl);
  mins[id] = mn;
  deltas[id] = dl;
}

__global__ void prefix_kernel(Geo g, const uint8_t* __restrict__ base, int p, uint8_t* __restrict__ out) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)g.rows * g.cols) return;
  out[id] = (uint8_t)load_code(g, base, (int)(id / g.cols), (int)(id % g.cols), p);
}

// Bit-exact dequantization: fmaf(bucket, step, min) rounds the exact value
// min + bucket*step once to f32, which equals float32 of the reference's
// float64 result (bucket*step is exact in f64).
__global__ void dequant_kernel(Geo g, const uint8_t* __restrict__ base, int p, float* __restrict__ out) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)g.rows * g.cols) return;
  const int r = (int)(id / g.cols), c = (int)(id % g.cols);
  float mn, dl;
  load_scale(g, base, r, c, &mn, &dl);
  out[id] = __fmaf_rn(bucket(load_code(g, base, r, c, p), p, g.p_max), dl, mn);
}

__global__ void gather_rows_kernel(Geo g, const uint8_t* __restrict__ base, const int32_t* __restrict__ ids, int n,
                                   const int32_t* __restrict__ p_dev, float* __restrict__ out) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)n * g.cols) return;
  int p = *p_dev;
  p = p < 1 ? 1 : (p > g.p_max ? g.p_max : p);
  const int i = (int)(id / g.cols), c = (int)(id % g.cols);
  int r = ids[i];
  r = r < 0 ? 0 : (r >= g.rows ? g.rows - 1 : r);
  float mn, dl;
  load_scale(g, base, r, c, &mn, &dl);
  out[id] = __fmaf_rn(bucket(load_code(g, base, r, c, p), p, g.p_max), dl, mn);
}

Geo geo_of(const pmpd_qtensor* t) {
  Geo g;
  g.rows = t->rows;
  g.cols = t->cols;
  g.gs = t->group_size;
  g.p_max = t->p_max;
  g.layout = t->layout;
  g.n = t->n;
  g.k = t->k;
  g.nt = t->n_tiles;
  g.kt = t->k_tiles;
  g.groups = t->groups;
  g.plane_bytes = t->plane_bytes;
  return g;
}

int check_tensor(const pmpd_qtensor* t) {
  if (!t || !t->data) return fail(PMPD_ERR_CONFIG, "null quantized tensor or data pointer");
  return PMPD_OK;
}

}  // namespace
}  // namespace pmpd

using namespace pmpd;

extern "C" {

int pmpd_version(int32_t* major, int32_t* minor) {
  if (major) *major = 0;
  if (minor) *minor = 1;
  return PMPD_OK;
}

const char* pmpd_last_error(void) { return last_error_slot().c_str(); }

int pmpd_qtensor_describe(int32_t rows, int32_t cols, int32_t group_size, int32_t p_max, int32_t layout,
                          pmpd_qtensor* out) {
  if (!out) return fail(PMPD_ERR_CONFIG, "null output descriptor");
  if (rows < 1 || cols < 1) return fail(PMPD_ERR_INPUT, "matrix shape must be positive, got %d x %d", rows, cols);
  if (p_max < 1 || p_max > 8) return fail(PMPD_ERR_CONFIG, "p_max must lie in [1, 8], got %d", p_max);
  if (group_size < 1) return fail(PMPD_ERR_CONFIG, "group_size must be >= 1, got %d", group_size);
  if (layout != PMPD_LAYOUT_REF && !is_tiled(layout)) return fail(PMPD_ERR_CONFIG, "unknown layout %d", layout);
  if (is_tiled(layout) && (group_size % kTile != 0 || p_max > 4))
    return fail(PMPD_ERR_CONFIG, "tiled layouts need group_size %% 64 == 0 and p_max <= 4 (got %d, %d)", group_size,
                p_max);
  pmpd_qtensor t{};
  t.rows = rows;
  t.cols = cols;
  t.group_size = group_size;
  t.p_max = p_max;
  t.layout = layout;
  t.groups = (cols + group_size - 1) / group_size;
  if (layout == PMPD_LAYOUT_KN) {
    t.n = cols;
    t.k = rows;
  } else {
    t.n = rows;
    t.k = cols;
  }
  if (is_tiled(layout)) {
    t.n_tiles = (t.n + kTile - 1) / kTile;
    t.k_tiles = (t.k + kTile - 1) / kTile;
    t.plane_bytes = (int64_t)t.n_tiles * t.k_tiles * kTilePlaneBytes;
    t.scale_bytes = (int64_t)t.n_tiles * t.k_tiles * kTileScaleBytes;
    t.aux_bytes = layout == PMPD_LAYOUT_KN ? ((int64_t)t.n_tiles * 4 + 255) / 256 * 256 : 0;
  } else {
    t.n_tiles = t.k_tiles = 0;
    t.plane_bytes = ((int64_t)rows * cols + 7) / 8;
    t.plane_bytes = (t.plane_bytes + 15) / 16 * 16;  // keep the scale region 16-byte aligned
    t.scale_bytes = 2LL * rows * t.groups * 4;
  }
  t.total_bytes = (int64_t)p_max * t.plane_bytes + t.scale_bytes + t.aux_bytes;
  t.data = out->data;
  *out = t;
  return PMPD_OK;
}

int pmpd_quantize(const void* w_dev, int32_t dtype, int32_t rows, int32_t cols, int32_t p_max, int32_t group_size,
                  uint8_t* codes, uint8_t* planes, float* mins, float* deltas, int32_t* nonfinite, void* stream) {
  if (p_max < 1 || p_max > 8) return fail(PMPD_ERR_CONFIG, "p_max must lie in [1, 8], got %d", p_max);
  if (group_size < 1) return fail(PMPD_ERR_CONFIG, "group_size must be >= 1, got %d", group_size);
  if (rows < 1 || cols < 1) return fail(PMPD_ERR_INPUT, "expected a non-empty 2-D weight matrix");
  const int groups = (cols + group_size - 1) / group_size;
  const int64_t ng = (int64_t)rows * groups;
  cudaStream_t s = as_stream(stream);
  const int levels = (1 << p_max) - 1;
  if (dtype == PMPD_DTYPE_F32)
    quantize_kernel<float><<<blocks_for(ng), kThreads, 0, s>>>((const float*)w_dev, rows, cols, group_size, groups,
                                                                levels, codes, mins, deltas, nonfinite);
  else if (dtype == PMPD_DTYPE_F64)
    quantize_kernel<double><<<blocks_for(ng), kThreads, 0, s>>>((const double*)w_dev, rows, cols, group_size, groups,
                                                                 levels, codes, mins, deltas, nonfinite);
  else if (dtype == PMPD_DTYPE_F16)
    quantize_kernel<__half><<<blocks_for(ng), kThreads, 0, s>>>((const __half*)w_dev, rows, cols, group_size, groups,
                                                                 levels, codes, mins, deltas, nonfinite);
  else
    return fail(PMPD_ERR_CONFIG, "unsupported weight dtype %d", dtype);
  const int64_t n = (int64_t)rows * cols, pb = (n + 7) / 8;
  planes_from_codes_kernel<<<blocks_for(pb * p_max), kThreads, 0, s>>>(codes, n, p_max, pb, planes);
  return check_launch("pmpd_quantize");
}

int pmpd_planes_from_codes(const uint8_t* codes, int32_t rows, int32_t cols, int32_t p_max, uint8_t* planes,
                           void* stream) {
  if (p_max < 1 || p_max > 8) return fail(PMPD_ERR_CONFIG, "p_max must lie in [1, 8], got %d", p_max);
  if (rows < 1 || cols < 1) return fail(PMPD_ERR_INPUT, "codes must be a non-empty 2-D array");
  const int64_t n = (int64_t)rows * cols, pb = (n + 7) / 8;
  planes_from_codes_kernel<<<blocks_for(pb * p_max), kThreads, 0, as_stream(stream)>>>(codes, n, p_max, pb, planes);
  return check_launch("pmpd_planes_from_codes");
}

int pmpd_pack(const pmpd_qtensor* t, const uint8_t* ref_planes, const float* mins, const float* deltas, void* stream) {
  if (int e = check_tensor(t)) return e;
  cudaStream_t s = as_stream(stream);
  const Geo g = geo_of(t);
  const int64_t ref_pb = ((int64_t)t->rows * t->cols + 7) / 8;
  uint8_t* base = static_cast<uint8_t*>(t->data);
  if (t->layout == PMPD_LAYOUT_REF) {
    for (int j = 0; j < t->p_max; ++j)
      cudaMemcpyAsync(base + (int64_t)j * t->plane_bytes, ref_planes + (int64_t)j * ref_pb, ref_pb,
                      cudaMemcpyDeviceToDevice, s);
    const int64_t sb = (int64_t)t->rows * t->groups * 4;
    uint8_t* scales = base + (int64_t)t->p_max * t->plane_bytes;
    cudaMemcpyAsync(scales, mins, sb, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(scales + sb, deltas, sb, cudaMemcpyDeviceToDevice, s);
    return check_launch("pmpd_pack(ref)");
  }
  const int64_t words = t->plane_bytes / 4 * t->p_max;
  pack_planes_kernel<<<blocks_for(words), kThreads, 0, s>>>(g, ref_planes, ref_pb, reinterpret_cast<uint32_t*>(base));
  const int64_t nsc = (int64_t)t->n_tiles * t->k_tiles * 128;
  pack_scales_kernel<<<blocks_for(nsc), kThreads, 0, s>>>(
      g, mins, deltas, reinterpret_cast<float*>(base + (int64_t)t->p_max * t->plane_bytes));
  if (t->layout == PMPD_LAYOUT_KN)
    pack_aux_kernel<<<t->n_tiles, kThreads, 0, s>>>(
        g, deltas, reinterpret_cast<float*>(base + (int64_t)t->p_max * t->plane_bytes + t->scale_bytes));
  return check_launch("pmpd_pack");
}

int pmpd_unpack(const pmpd_qtensor* t, uint8_t* ref_planes, float* mins, float* deltas, void* stream) {
  if (int e = check_tensor(t)) return e;
  cudaStream_t s = as_stream(stream);
  const Geo g = geo_of(t);
  const int64_t ref_pb = ((int64_t)t->rows * t->cols + 7) / 8;
  const uint8_t* base = static_cast<const uint8_t*>(t->data);
  if (t->layout == PMPD_LAYOUT_REF) {
    for (int j = 0; j < t->p_max; ++j)
      cudaMemcpyAsync(ref_planes + (int64_t)j * ref_pb, base + (int64_t)j * t->plane_bytes, ref_pb,
                      cudaMemcpyDeviceToDevice, s);
  } else {
    unpack_planes_kernel<<<blocks_for(ref_pb * t->p_max), kThreads, 0, s>>>(g, base, ref_pb, ref_planes);
  }
  unpack_scales_kernel<<<blocks_for((int64_t)t->rows * t->groups), kThreads, 0, s>>>(g, base, mins, deltas);
  return check_launch("pmpd_unpack");
}

int pmpd_prefix_codes(const pmpd_qtensor* t, int32_t p, uint8_t* codes, void* stream) {
  if (int e = check_tensor(t)) return e;
  if (p < 1 || p > t->p_max) return fail(PMPD_ERR_CONFIG, "precision %d outside [1, %d]", p, t->p_max);
  const int64_t n = (int64_t)t->rows * t->cols;
  prefix_kernel<<<blocks_for(n), kThreads, 0, as_stream(stream)>>>(geo_of(t), (const uint8_t*)t->data, p, codes);
  return check_launch("pmpd_prefix_codes");
}

int pmpd_dequant(const pmpd_qtensor* t, int32_t p, float* out, void* stream) {
  if (int e = check_tensor(t)) return e;
  if (p < 1 || p > t->p_max) return fail(PMPD_ERR_CONFIG, "precision %d outside [1, %d]", p, t->p_max);
  const int64_t n = (int64_t)t->rows * t->cols;
  dequant_kernel<<<blocks_for(n), kThreads, 0, as_stream(stream)>>>(geo_of(t), (const uint8_t*)t->data, p, out);
  return check_launch("pmpd_dequant");
}

int pmpd_gather_rows(const pmpd_qtensor* t, const int32_t* ids, int32_t n, const int32_t* p_dev, float* out,
                     void* stream) {
  if (int e = check_tensor(t)) return e;
  if (n < 1) return fail(PMPD_ERR_INPUT, "gather needs at least one row id");
  const int64_t cnt = (int64_t)n * t->cols;
  gather_rows_kernel<<<blocks_for(cnt), kThreads, 0, as_stream(stream)>>>(geo_of(t), (const uint8_t*)t->data, ids, n,
                                                                          p_dev, out);
  return check_launch("pmpd_gather_rows");
}

}  // extern "C"

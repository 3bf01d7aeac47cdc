// Decoder glue kernels of the device model (everything between the quantized
// linear layers) and the device-side learned switch predictor.
//
// Reference: pkg/src/pmpd/tinylm.py:293-368 (_rmsnorm 293-295, _silu 298,
// _softmax 302-305, _rope_tables/_apply_rope 308-319, attention 349-358,
// residual adds 359/364), sample() greedy argmax 422-429, and
// learnsched.py:118-160 (_pool_forward + predict_schedule).
//
// Conventions: residual stream f32, GEMV inputs f16, KV cache f16 (post-RoPE K
// and V rows, flattened heads, as KVCache stores them, tinylm.py:272-286).
// Positions come from a device counter (*T_dev = tokens already cached), so
// a whole decode step can be replayed as a CUDA graph without host syncs.
#include <cuda_fp16.h>
#include <float.h>

#include "pmpd_common.cuh"
#include "pmpd_internal.h"

namespace pmpd {
namespace {

constexpr int kBlock = 256;

PMPD_DEV float block_sum(float v, float* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float r = 0.f;
  for (int i = 0; i < nw; ++i) r += sh[i];
  return r;
}

PMPD_DEV float block_max(float v, float* sh) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float r = -FLT_MAX;
  for (int i = 0; i < nw; ++i) r = fmaxf(r, sh[i]);
  return r;
}

// out[m][i] = f16(x[m][i] / sqrt(mean(x[m]^2) + eps) * gain[i])   (tinylm.py:293-295)
__global__ void rmsnorm_kernel(const float* __restrict__ x, int ldx, const float* __restrict__ gain, int d, float eps,
                               __half* __restrict__ out, int ldo) {
  __shared__ float sh[32];
  const float* xr = x + (int64_t)blockIdx.x * ldx;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(xr[i], xr[i], ss);
  ss = block_sum(ss, sh);
  const float inv = rsqrtf(ss / (float)d + eps);
  __half* o = out + (int64_t)blockIdx.x * ldo;
  for (int i = threadIdx.x; i < d; i += blockDim.x) o[i] = __float2half(xr[i] * inv * gain[i]);
}

// Rotate-half RoPE on q and k of m new tokens at positions T+i (tinylm.py:308-319,344-347);
// q -> q_out (f32), post-RoPE k and raw v -> KV cache rows T+i (f16).
// cos/sin: [max_ctx][d_head/2] tables computed in float64 on the host.
__global__ void rope_kv_kernel(const float* __restrict__ qkv, int ldq, int d, int dh, const float* __restrict__ cos_t,
                               const float* __restrict__ sin_t, const int32_t* __restrict__ T_dev, int max_ctx,
                               float* __restrict__ q_out, __half* __restrict__ kc, __half* __restrict__ vc) {
  const int i = blockIdx.x;  // token
  const int pos = *T_dev + i;
  if (pos >= max_ctx) return;
  const float* row = qkv + (int64_t)i * ldq;
  const int half = dh >> 1;
  for (int e = threadIdx.x; e < d / 2; e += blockDim.x) {
    const int h = e / half, j = e - h * half;
    const float c = cos_t[(int64_t)pos * half + j], s = sin_t[(int64_t)pos * half + j];
    const int a = h * dh + j, b = a + half;
    const float q1 = row[a], q2 = row[b];
    q_out[(int64_t)i * d + a] = q1 * c - q2 * s;
    q_out[(int64_t)i * d + b] = q2 * c + q1 * s;
    const float k1 = row[d + a], k2 = row[d + b];
    kc[(int64_t)pos * d + a] = __float2half(k1 * c - k2 * s);
    kc[(int64_t)pos * d + b] = __float2half(k2 * c + k1 * s);
    vc[(int64_t)pos * d + a] = __float2half(row[2 * d + a]);
    vc[(int64_t)pos * d + b] = __float2half(row[2 * d + b]);
  }
}

// Causal multi-head attention of m new queries over the cache (tinylm.py:349-358).
// One block per (query i, head h); query i attends to positions 0..T+i.
// Scores and softmax in f32; ctx -> out f16 [m][d].
__global__ void attention_kernel(const float* __restrict__ q, int d, int dh, const __half* __restrict__ kc,
                                 const __half* __restrict__ vc, const int32_t* __restrict__ T_dev, int max_ctx,
                                 float scale, __half* __restrict__ out) {
  extern __shared__ float sm[];  // [max_ctx] scores + [dh] q + 32 scratch
  float* sc = sm;
  float* qs = sm + max_ctx;
  float* red = qs + dh;
  const int i = blockIdx.x, h = blockIdx.y;
  const int L = min(*T_dev + i + 1, max_ctx);
  for (int e = threadIdx.x; e < dh; e += blockDim.x) qs[e] = q[(int64_t)i * d + h * dh + e];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // scores: one warp per key row, lanes over the head dim
  for (int t = warp; t < L; t += nw) {
    const __half* kr = kc + (int64_t)t * d + h * dh;
    float acc = 0.f;
    for (int e = lane; e < dh; e += 32) acc = fmaf(qs[e], __half2float(kr[e]), acc);
    acc = warp_sum(acc);
    if (lane == 0) sc[t] = acc * scale;
  }
  __syncthreads();
  float mx = -FLT_MAX;
  for (int t = threadIdx.x; t < L; t += blockDim.x) mx = fmaxf(mx, sc[t]);
  mx = block_max(mx, red);
  float sum = 0.f;
  for (int t = threadIdx.x; t < L; t += blockDim.x) {
    const float e = __expf(sc[t] - mx);
    sc[t] = e;
    sum += e;
  }
  sum = block_sum(sum, red);
  const float inv = 1.f / sum;
  __syncthreads();
  // ctx[e] = sum_t a_t V[t][h*dh+e]
  for (int e = threadIdx.x; e < dh; e += blockDim.x) {
    float acc = 0.f;
    const __half* vr = vc + h * dh + e;
    for (int t = 0; t < L; ++t) acc = fmaf(sc[t], __half2float(vr[(int64_t)t * d]), acc);
    out[(int64_t)i * d + h * dh + e] = __float2half(acc * inv);
  }
}

// out[m][j] = f16(silu(u[m][j]) * u[m][ff + j])   (tinylm.py:298,362-364)
__global__ void silu_mul_kernel(const float* __restrict__ u, int ldu, int ff, int m, __half* __restrict__ out,
                                int ldo) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)m * ff) return;
  const int r = (int)(id / ff), j = (int)(id % ff);
  const float g = u[(int64_t)r * ldu + j], up = u[(int64_t)r * ldu + ff + j];
  out[(int64_t)r * ldo + j] = __float2half(g / (1.f + __expf(-g)) * up);
}

// Greedy sampling: argmax with the lowest index on ties (tinylm.py:428-429, np.argmax).
// Non-finite logits raise InputError in the reference; here they set *bad.
__global__ void argmax_kernel(const float* __restrict__ logits, int ld, int V, int32_t* __restrict__ out,
                              int32_t* __restrict__ bad) {
  __shared__ float sv[32];
  __shared__ int si[32];
  const float* row = logits + (int64_t)blockIdx.x * ld;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  bool nonfinite = false;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const float v = row[j];
    nonfinite |= !isfinite(v);
    if (v > best || (v == best && j < bi)) {
      best = v;
      bi = j;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  if (nonfinite && bad) *bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b0 = sv[0];
    int i0 = si[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (sv[k] > b0 || (sv[k] == b0 && si[k] < i0)) {
        b0 = sv[k];
        i0 = si[k];
      }
    out[blockIdx.x] = i0;
  }
}

__global__ void add_i32_kernel(int32_t* p, int v) { *p += v; }

// dst[*idx][0..n) = src[0..n) when *idx < capacity (per-step logits history).
__global__ void store_row_kernel(const float* __restrict__ src, float* __restrict__ dst, const int32_t* __restrict__ idx,
                                 int n, int capacity) {
  const int r = *idx;
  if (r >= capacity) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    dst[(int64_t)r * n + j] = src[j];
}

// Token bookkeeping of one greedy decode step, all on device:
//   tokens[*n] = argmax already written to *cur; n += 1; T += 1 (the cache grew by one row).
__global__ void push_token_kernel(const int32_t* __restrict__ cur, int32_t* __restrict__ tokens,
                                  int32_t* __restrict__ n, int32_t* __restrict__ T, int capacity) {
  const int k = *n;
  if (k < capacity) tokens[k] = *cur;
  *n = k + 1;
  if (T) *T += 1;
}

// ------------------------------------------------------------------ learned scheduler
// s = K q / sqrt(d_k); a = softmax(s); pooled = a V; h = relu(W1 pooled + b1);
// logits = W2 h + b2; cls = argmax (lowest on ties); switch = grid[cls]
// -> schedule table {p_high: 0, p_low: switch} (learnsched.py:118-125,151-160).
// One block; K/V are the cache rows 0..T-1 of the feature block (f16).
__global__ void learned_predict_kernel(const __half* __restrict__ K, const __half* __restrict__ V, int ldkv,
                                       const int32_t* __restrict__ T_dev, int dk, int dv, int hidden, int ncls,
                                       const float* __restrict__ qv, const float* __restrict__ w1,
                                       const float* __restrict__ b1, const float* __restrict__ w2,
                                       const float* __restrict__ b2, const int32_t* __restrict__ grid_pts,
                                       int p_high, int p_low, int32_t* __restrict__ sched, float* __restrict__ dbg) {
  extern __shared__ float sm[];  // [T] scores | [dv] pooled | [hidden] h | 32
  const int T = *T_dev;
  float* sc = sm;
  float* pooled = sc + T;
  float* hid = pooled + dv;
  float* red = hid + hidden;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const float inv_sqrt = rsqrtf((float)dk);
  for (int t = warp; t < T; t += nw) {
    float acc = 0.f;
    for (int e = lane; e < dk; e += 32) acc = fmaf(__half2float(K[(int64_t)t * ldkv + e]), qv[e], acc);
    acc = warp_sum(acc);
    if (lane == 0) sc[t] = acc * inv_sqrt;
  }
  __syncthreads();
  float mx = -FLT_MAX;
  for (int t = threadIdx.x; t < T; t += blockDim.x) mx = fmaxf(mx, sc[t]);
  mx = block_max(mx, red);
  float sum = 0.f;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const float e = __expf(sc[t] - mx);
    sc[t] = e;
    sum += e;
  }
  sum = block_sum(sum, red);
  const float inv = 1.f / sum;
  __syncthreads();
  for (int e = threadIdx.x; e < dv; e += blockDim.x) {
    float acc = 0.f;
    for (int t = 0; t < T; ++t) acc = fmaf(sc[t], __half2float(V[(int64_t)t * ldkv + e]), acc);
    pooled[e] = acc * inv;
  }
  __syncthreads();
  for (int j = warp; j < hidden; j += nw) {
    float acc = 0.f;
    for (int e = lane; e < dv; e += 32) acc = fmaf(w1[(int64_t)j * dv + e], pooled[e], acc);
    acc = warp_sum(acc);
    if (lane == 0) hid[j] = fmaxf(acc + b1[j], 0.f);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int best_i = 0;
    float best = -INFINITY;
    for (int c = 0; c < ncls; ++c) {
      float acc = b2[c];
      for (int j = 0; j < hidden; ++j) acc = fmaf(w2[(int64_t)c * hidden + j], hid[j], acc);
      if (dbg) dbg[c] = acc;
      if (acc > best) {
        best = acc;
        best_i = c;
      }
    }
    // two-phase schedule, fixed-capacity table layout (p, st) pairs, unused p = 0
    sched[0] = p_high;
    sched[1] = 0;
    sched[2] = p_low;
    sched[3] = grid_pts[best_i];
    for (int q = 4; q < 16; ++q) sched[q] = 0;
  }
}

}  // namespace
}  // namespace pmpd

using namespace pmpd;

extern "C" {

int pmpd_rmsnorm(const float* x, int32_t ldx, const float* gain, int32_t m, int32_t d, float eps, void* out,
                 int32_t ldo, void* stream) {
  if (m < 1 || d < 1) return fail(PMPD_ERR_INPUT, "rmsnorm needs m, d >= 1");
  rmsnorm_kernel<<<m, kBlock, 0, as_stream(stream)>>>(x, ldx, gain, d, eps, (__half*)out, ldo);
  return check_launch("pmpd_rmsnorm");
}

int pmpd_rope_kv(const float* qkv, int32_t ldq, int32_t m, int32_t d, int32_t d_head, const float* cos_t,
                 const float* sin_t, const int32_t* T_dev, int32_t max_ctx, float* q_out, void* k_cache,
                 void* v_cache, void* stream) {
  if (d_head % 2 || d % d_head) return fail(PMPD_ERR_CONFIG, "bad head geometry");
  rope_kv_kernel<<<m, kBlock, 0, as_stream(stream)>>>(qkv, ldq, d, d_head, cos_t, sin_t, T_dev, max_ctx, q_out,
                                                      (__half*)k_cache, (__half*)v_cache);
  return check_launch("pmpd_rope_kv");
}

int pmpd_attention(const float* q, int32_t m, int32_t d, int32_t d_head, const void* k_cache, const void* v_cache,
                   const int32_t* T_dev, int32_t max_ctx, float scale, void* out, void* stream) {
  if (d % d_head) return fail(PMPD_ERR_CONFIG, "bad head geometry");
  const size_t smem = (size_t)(max_ctx + d_head + 32) * sizeof(float);
  if (smem > 200 * 1024) return fail(PMPD_ERR_CONFIG, "context too long for the attention kernel");
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  attention_kernel<<<dim3(m, d / d_head), kBlock, smem, as_stream(stream)>>>(
      q, d, d_head, (const __half*)k_cache, (const __half*)v_cache, T_dev, max_ctx, scale, (__half*)out);
  return check_launch("pmpd_attention");
}

int pmpd_silu_mul(const float* u, int32_t ldu, int32_t m, int32_t ff, void* out, int32_t ldo, void* stream) {
  const int64_t n = (int64_t)m * ff;
  silu_mul_kernel<<<(unsigned)((n + kBlock - 1) / kBlock), kBlock, 0, as_stream(stream)>>>(u, ldu, ff, m,
                                                                                          (__half*)out, ldo);
  return check_launch("pmpd_silu_mul");
}

int pmpd_argmax(const float* logits, int32_t ld, int32_t m, int32_t V, int32_t* out, int32_t* bad, void* stream) {
  argmax_kernel<<<m, 1024, 0, as_stream(stream)>>>(logits, ld, V, out, bad);
  return check_launch("pmpd_argmax");
}

int pmpd_add_i32(int32_t* p, int32_t v, void* stream) {
  add_i32_kernel<<<1, 1, 0, as_stream(stream)>>>(p, v);
  return check_launch("pmpd_add_i32");
}

int pmpd_store_row(const float* src, float* dst, const int32_t* idx, int32_t n, int32_t capacity, void* stream) {
  store_row_kernel<<<(n + 1023) / 1024 < 64 ? (n + 1023) / 1024 : 64, 1024, 0, as_stream(stream)>>>(src, dst, idx, n,
                                                                                                   capacity);
  return check_launch("pmpd_store_row");
}

int pmpd_push_token(const int32_t* cur, int32_t* tokens, int32_t* n, int32_t* T, int32_t capacity, void* stream) {
  push_token_kernel<<<1, 1, 0, as_stream(stream)>>>(cur, tokens, n, T, capacity);
  return check_launch("pmpd_push_token");
}

int pmpd_learned_predict(const void* K, const void* V, int32_t ldkv, const int32_t* T_dev, int32_t max_T, int32_t dk,
                         int32_t dv, int32_t hidden, int32_t ncls, const float* q, const float* w1, const float* b1,
                         const float* w2, const float* b2, const int32_t* grid_pts, int32_t p_high, int32_t p_low,
                         int32_t* sched_dev, float* dbg_logits, void* stream) {
  if (ncls < 1 || hidden < 1) return fail(PMPD_ERR_CONFIG, "bad scheduler net shape");
  const size_t smem = (size_t)(max_T + dv + hidden + 32) * sizeof(float);
  if (smem > 200 * 1024) return fail(PMPD_ERR_CONFIG, "scheduler net too large for one block");
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(learned_predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  learned_predict_kernel<<<1, 1024, smem, as_stream(stream)>>>((const __half*)K, (const __half*)V, ldkv, T_dev, dk, dv,
                                                               hidden, ncls, q, w1, b1, w2, b2, grid_pts, p_high,
                                                               p_low, sched_dev, dbg_logits);
  return check_launch("pmpd_learned_predict");
}

}  // extern "C"

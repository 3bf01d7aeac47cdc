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
#include <cooperative_groups.h>
#include <float.h>
#include <stdlib.h>

#include "pmpd_common.cuh"
#include "pmpd_internal.h"

namespace pmpd {
namespace cg = cooperative_groups;
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
  pdl_launch_dependents();  // a following PDL GEMV / GEMM may stream its weights meanwhile
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
                               float* __restrict__ q_out, __half* __restrict__ kc, __half* __restrict__ vc,
                               int vec2) {
  const int i = blockIdx.x;  // token
  const int pos = *T_dev + i;
  if (pos >= max_ctx) return;
  const float* row = qkv + (int64_t)i * ldq;
  const int half = dh >> 1;
  if (vec2) {
    // two adjacent rotation pairs (j, j + 1) per thread: float2 loads/stores, half2 cache writes
    for (int e = 2 * threadIdx.x; e < d / 2; e += 2 * blockDim.x) {
      const int h = e / half, j = e - h * half;
      const float2 c = *reinterpret_cast<const float2*>(cos_t + (int64_t)pos * half + j);
      const float2 s = *reinterpret_cast<const float2*>(sin_t + (int64_t)pos * half + j);
      const int a = h * dh + j, b = a + half;
      const float2 q1 = *reinterpret_cast<const float2*>(row + a), q2 = *reinterpret_cast<const float2*>(row + b);
      *reinterpret_cast<float2*>(q_out + (int64_t)i * d + a) = make_float2(q1.x * c.x - q2.x * s.x, q1.y * c.y - q2.y * s.y);
      *reinterpret_cast<float2*>(q_out + (int64_t)i * d + b) = make_float2(q2.x * c.x + q1.x * s.x, q2.y * c.y + q1.y * s.y);
      const float2 k1 = *reinterpret_cast<const float2*>(row + d + a), k2 = *reinterpret_cast<const float2*>(row + d + b);
      *reinterpret_cast<__half2*>(kc + (int64_t)pos * d + a) =
          __floats2half2_rn(k1.x * c.x - k2.x * s.x, k1.y * c.y - k2.y * s.y);
      *reinterpret_cast<__half2*>(kc + (int64_t)pos * d + b) =
          __floats2half2_rn(k2.x * c.x + k1.x * s.x, k2.y * c.y + k1.y * s.y);
      const float2 v1 = *reinterpret_cast<const float2*>(row + 2 * d + a), v2 = *reinterpret_cast<const float2*>(row + 2 * d + b);
      *reinterpret_cast<__half2*>(vc + (int64_t)pos * d + a) = __floats2half2_rn(v1.x, v1.y);
      *reinterpret_cast<__half2*>(vc + (int64_t)pos * d + b) = __floats2half2_rn(v2.x, v2.y);
    }
    return;
  }
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
  pdl_launch_dependents();  // a following PDL GEMV / GEMM may stream its weights meanwhile
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

// Split-context ("flash-decoding") attention for head dims 32*DPL: one thread-block
// cluster of kSplit CTAs per (query i, head h).  CTA r takes positions
// [r*ceil(L/kSplit), ...) and its warps stream K/V rows (lane l holds dims
// l*DPL..+DPL, so one row is one coalesced warp load) with an online softmax in
// registers.  Warp partials fold into a CTA partial (max, sum, acc[dh]) in
// shared memory; after a cluster barrier every CTA reads all kSplit partials
// over DSMEM and writes its dh/kSplit slice of the output.  Same math as
// attention_kernel (tinylm.py:349-358), re-associated: f32, exp via __expf.
constexpr int kSplit = 8;
constexpr int kAttnWarps = 4;
constexpr int kAttnUnroll = 4;

template <int DPL>
PMPD_DEV void load_row(const __half* __restrict__ p, float (&f)[DPL]) {
  if constexpr (DPL == 1) {
    f[0] = __half2float(*p);
  } else if constexpr (DPL == 2) {
    const float2 v = __half22float2(*reinterpret_cast<const __half2*>(p));
    f[0] = v.x;
    f[1] = v.y;
  } else if constexpr (DPL == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
  } else {
    static_assert(DPL == 8, "head dim must be 32, 64, 128 or 256");
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&w[j]));
      f[2 * j] = v.x;
      f[2 * j + 1] = v.y;
    }
  }
}

// ROPE (decode, one query): q comes raw from the q|k|v row `q` (ldq = its width) and is rotated
// here; the CTA whose split holds the new position also rotates k, and writes k and v into cache
// row T (f16, as rope_kv_kernel does) before reading it back in its loop.  RoPE pairs dim j with
// j + dh/2, which for every DPL sits in lane ^ 16 (tinylm.py:308-319,344-347).
template <int DPL, bool ROPE>
__global__ void __cluster_dims__(kSplit, 1, 1) __launch_bounds__(kAttnWarps * 32)
    attention_split_kernel(const float* __restrict__ q, int d, __half* __restrict__ kc, __half* __restrict__ vc,
                           const int32_t* __restrict__ T_dev, int max_ctx, float scale, __half* __restrict__ out,
                           const float* __restrict__ cos_t, const float* __restrict__ sin_t, int ldq = 0,
                           int64_t sstride = 0) {
  pdl_launch_dependents();  // the o GEMV (PDL) may stream its weights meanwhile
  constexpr int DH = 32 * DPL;
  __shared__ float w_ml[kAttnWarps][2];
  __shared__ float w_acc[kAttnWarps][DH];
  __shared__ float c_ml[2];
  __shared__ float c_acc[DH];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int qh = blockIdx.x / kSplit, H = d / DH;
  const int i = qh / H, h = qh - i * H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ROPE: i is a sequence (one new token each, its own cache at kc + i * sstride and length T_dev[i]);
  // otherwise i is the i-th of m causal queries over one cache
  const int Ti = ROPE ? T_dev[i] : *T_dev;
  const int L = ROPE ? min(Ti + 1, max_ctx) : min(Ti + i + 1, max_ctx);
  if constexpr (ROPE) {
    q += (int64_t)i * ldq;
    kc += (int64_t)i * sstride;
    vc += (int64_t)i * sstride;
  }
  const int chunk = (L + kSplit - 1) / kSplit;
  const int t0 = rank * chunk, t1 = min(L, t0 + chunk);

  float qr[DPL];
  if constexpr (!ROPE) {
#pragma unroll
    for (int j = 0; j < DPL; ++j) qr[j] = q[(int64_t)i * d + h * DH + lane * DPL + j];
  } else {
    // position T = L - 1 (the row being appended)
    constexpr int HALF = DH / 2;
    const int pos = L - 1;
    const bool first = lane < 16;
    float c[DPL], sn[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
      const int jj = (lane * DPL + j) % HALF;
      c[j] = cos_t[(int64_t)pos * HALF + jj];
      sn[j] = sin_t[(int64_t)pos * HALF + jj];
    }
    auto rot = [&](const float* src, float (&dst)[DPL]) {
#pragma unroll
      for (int j = 0; j < DPL; ++j) {
        const float a = src[h * DH + lane * DPL + j];
        const float b = __shfl_xor_sync(0xffffffffu, a, 16);  // partner dim j +- HALF
        dst[j] = first ? a * c[j] - b * sn[j] : a * c[j] + b * sn[j];
      }
    };
    rot(q, qr);
    if (Ti < max_ctx && pos >= t0 && pos < t1 && warp == 0) {
      float kr[DPL];
      rot(q + d, kr);
#pragma unroll
      for (int j = 0; j < DPL; ++j) {
        kc[(int64_t)pos * d + h * DH + lane * DPL + j] = __float2half(kr[j]);
        vc[(int64_t)pos * d + h * DH + lane * DPL + j] = __float2half(q[2 * d + h * DH + lane * DPL + j]);
      }
    }
    __syncthreads();  // the appended row is read below by every warp of this CTA
  }
  const __half* kb = kc + h * DH + lane * DPL;
  const __half* vb = vc + h * DH + lane * DPL;
  float m = -INFINITY, l = 0.f, acc[DPL];
#pragma unroll
  for (int j = 0; j < DPL; ++j) acc[j] = 0.f;

  for (int tb = t0 + warp; tb < t1; tb += kAttnWarps * kAttnUnroll) {
    float kf[kAttnUnroll][DPL], vf[kAttnUnroll][DPL], s[kAttnUnroll];
#pragma unroll
    for (int u = 0; u < kAttnUnroll; ++u) {
      const int t = tb + u * kAttnWarps;
      if (t < t1) {
        load_row<DPL>(kb + (int64_t)t * d, kf[u]);
        load_row<DPL>(vb + (int64_t)t * d, vf[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kAttnUnroll; ++u) {
      float a = 0.f;
#pragma unroll
      for (int j = 0; j < DPL; ++j) a = fmaf(qr[j], kf[u][j], a);
      s[u] = a;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < kAttnUnroll; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
#pragma unroll
    for (int u = 0; u < kAttnUnroll; ++u) {
      if (tb + u * kAttnWarps < t1) {
        const float sc = s[u] * scale;
        const float mn = fmaxf(m, sc);
        const float corr = __expf(m - mn), pe = __expf(sc - mn);
        l = fmaf(l, corr, pe);
#pragma unroll
        for (int j = 0; j < DPL; ++j) acc[j] = fmaf(acc[j], corr, pe * vf[u][j]);
        m = mn;
      }
    }
  }
  if (lane == 0) {
    w_ml[warp][0] = m;
    w_ml[warp][1] = l;
  }
#pragma unroll
  for (int j = 0; j < DPL; ++j) w_acc[warp][lane * DPL + j] = acc[j];
  __syncthreads();
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, w_ml[w][0]);
  float wt[kAttnWarps], lc = 0.f;
#pragma unroll
  for (int w = 0; w < kAttnWarps; ++w) {
    wt[w] = w_ml[w][0] == -INFINITY ? 0.f : __expf(w_ml[w][0] - M);
    lc = fmaf(w_ml[w][1], wt[w], lc);
  }
  for (int e = threadIdx.x; e < DH; e += kAttnWarps * 32) {
    float a = 0.f;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) a = fmaf(w_acc[w][e], wt[w], a);
    c_acc[e] = a;
  }
  if (threadIdx.x == 0) {
    c_ml[0] = M;
    c_ml[1] = lc;
  }
  cl.sync();
  // combine: this CTA writes dims [rank*DH/kSplit, (rank+1)*DH/kSplit)
  constexpr int SL = DH / kSplit;
  if (threadIdx.x < SL) {
    float Mg = -INFINITY;
    float rm[kSplit], rl[kSplit];
#pragma unroll
    for (int r = 0; r < kSplit; ++r) {
      const float* ml = cl.map_shared_rank(c_ml, r);
      rm[r] = ml[0];
      rl[r] = ml[1];
      Mg = fmaxf(Mg, rm[r]);
    }
    const int e = rank * SL + threadIdx.x;
    float num = 0.f, den = 0.f;
#pragma unroll
    for (int r = 0; r < kSplit; ++r) {
      const float wr = rm[r] == -INFINITY ? 0.f : __expf(rm[r] - Mg);
      den = fmaf(rl[r], wr, den);
      num = fmaf(cl.map_shared_rank(c_acc, r)[e], wr, num);
    }
    out[(int64_t)i * d + h * DH + e] = __float2half(num / den);
  }
  cl.sync();  // partials stay readable until every CTA of the cluster has combined
}

// out[m][i] = f16(x[m][i] * rsqrt(mean(x[m]^2) + eps) * gain[i]) with the row held in
// registers: R float4 per thread, one read of x (tinylm.py:293-295).
template <int R>
__global__ void __launch_bounds__(512) rmsnorm_vec_kernel(const float* __restrict__ x, int ldx,
                                                         const float* __restrict__ gain, int d, float eps,
                                                         __half* __restrict__ out, int ldo) {
  pdl_launch_dependents();  // a following PDL GEMV / GEMM may stream its weights meanwhile
  __shared__ float sh[32];
  const float4* xr = reinterpret_cast<const float4*>(x + (int64_t)blockIdx.x * ldx);
  const int n4 = d >> 2;
  float4 v[R];
  float ss = 0.f;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int j = threadIdx.x + r * blockDim.x;
    v[r] = j < n4 ? xr[j] : make_float4(0.f, 0.f, 0.f, 0.f);
    ss = fmaf(v[r].x, v[r].x, fmaf(v[r].y, v[r].y, fmaf(v[r].z, v[r].z, fmaf(v[r].w, v[r].w, ss))));
  }
  ss = block_sum(ss, sh);
  const float inv = rsqrtf(ss / (float)d + eps);
  uint2* o = reinterpret_cast<uint2*>(out + (int64_t)blockIdx.x * ldo);
  const float4* g4 = reinterpret_cast<const float4*>(gain);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int j = threadIdx.x + r * blockDim.x;
    if (j < n4) {
      const float4 g = g4[j];
      const __half2 a = __floats2half2_rn(v[r].x * inv * g.x, v[r].y * inv * g.y);
      const __half2 b = __floats2half2_rn(v[r].z * inv * g.z, v[r].w * inv * g.w);
      uint2 u;
      u.x = *reinterpret_cast<const uint32_t*>(&a);
      u.y = *reinterpret_cast<const uint32_t*>(&b);
      o[j] = u;
    }
  }
}

// out[m][j] = f16(silu(u[m][j]) * u[m][ff + j])   (tinylm.py:298,362-364)
// One row per blockIdx.y, 4 consecutive channels per thread (float4 loads, half2 stores when the
// row strides allow it; no per-element integer division).
PMPD_DEV float silu_times(float g, float up) { return g / (1.f + __expf(-g)) * up; }

__global__ void silu_mul_kernel(const float* __restrict__ u, int ldu, int ff, int m, __half* __restrict__ out,
                                int ldo, int vec) {
  pdl_launch_dependents();  // a following PDL GEMV / GEMM may stream its weights meanwhile
  const int r = blockIdx.y;
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (r >= m || j0 >= ff) return;
  const float* ur = u + (int64_t)r * ldu;
  __half* orow = out + (int64_t)r * ldo;
  if (vec && j0 + 4 <= ff) {
    const float4 g = *reinterpret_cast<const float4*>(ur + j0), up = *reinterpret_cast<const float4*>(ur + ff + j0);
    *reinterpret_cast<__half2*>(orow + j0) = __floats2half2_rn(silu_times(g.x, up.x), silu_times(g.y, up.y));
    *reinterpret_cast<__half2*>(orow + j0 + 2) = __floats2half2_rn(silu_times(g.z, up.z), silu_times(g.w, up.w));
  } else {
    for (int j = j0; j < j0 + 4 && j < ff; ++j) orow[j] = __float2half(silu_times(ur[j], ur[ff + j]));
  }
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
  const bool vec = d % 4 == 0 && ldx % 4 == 0 && ldo % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(gain) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 7) == 0;
  if (vec && d <= 128 * 4) {
    rmsnorm_vec_kernel<1><<<m, 128, 0, as_stream(stream)>>>(x, ldx, gain, d, eps, (__half*)out, ldo);
  } else if (vec && d <= 512 * 4 * 4) {
    rmsnorm_vec_kernel<4><<<m, 512, 0, as_stream(stream)>>>(x, ldx, gain, d, eps, (__half*)out, ldo);
  } else {
    rmsnorm_kernel<<<m, kBlock, 0, as_stream(stream)>>>(x, ldx, gain, d, eps, (__half*)out, ldo);
  }
  return check_launch("pmpd_rmsnorm");
}

int pmpd_rope_kv(const float* qkv, int32_t ldq, int32_t m, int32_t d, int32_t d_head, const float* cos_t,
                 const float* sin_t, const int32_t* T_dev, int32_t max_ctx, float* q_out, void* k_cache,
                 void* v_cache, void* stream) {
  if (d_head % 2 || d % d_head) return fail(PMPD_ERR_CONFIG, "bad head geometry");
  // float2 / half2 path: rotation pairs come in adjacent twos (d_head % 4 == 0) and every row is 8-byte aligned
  const int vec2 = d_head % 4 == 0 && ldq % 2 == 0 && d % 2 == 0 && (reinterpret_cast<uintptr_t>(qkv) & 7) == 0 &&
                   (reinterpret_cast<uintptr_t>(q_out) & 7) == 0 && (reinterpret_cast<uintptr_t>(cos_t) & 7) == 0 &&
                   (reinterpret_cast<uintptr_t>(sin_t) & 7) == 0 && (reinterpret_cast<uintptr_t>(k_cache) & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(v_cache) & 3) == 0;
  rope_kv_kernel<<<m, kBlock, 0, as_stream(stream)>>>(qkv, ldq, d, d_head, cos_t, sin_t, T_dev, max_ctx, q_out,
                                                      (__half*)k_cache, (__half*)v_cache, vec2);
  return check_launch("pmpd_rope_kv");
}

int pmpd_attention(const float* q, int32_t m, int32_t d, int32_t d_head, const void* k_cache, const void* v_cache,
                   const int32_t* T_dev, int32_t max_ctx, float scale, void* out, void* stream) {
  if (d % d_head) return fail(PMPD_ERR_CONFIG, "bad head geometry");
  const bool al = (reinterpret_cast<uintptr_t>(k_cache) & 15) == 0 && (reinterpret_cast<uintptr_t>(v_cache) & 15) == 0;
  static const bool generic = getenv("PMPD_ATTN_GENERIC") != nullptr;  // diagnostics: force attention_kernel
  if (al && m >= 1 && !generic) {
    const dim3 grid((unsigned)(m * (d / d_head) * kSplit));
    const auto kc = (__half*)const_cast<void*>(k_cache);
    const auto vc = (__half*)const_cast<void*>(v_cache);
    switch (d_head) {
      case 32:
        attention_split_kernel<1, false><<<grid, kAttnWarps * 32, 0, as_stream(stream)>>>(
            q, d, kc, vc, T_dev, max_ctx, scale, (__half*)out, nullptr, nullptr);
        return check_launch("pmpd_attention");
      case 64:
        attention_split_kernel<2, false><<<grid, kAttnWarps * 32, 0, as_stream(stream)>>>(
            q, d, kc, vc, T_dev, max_ctx, scale, (__half*)out, nullptr, nullptr);
        return check_launch("pmpd_attention");
      case 128:
        attention_split_kernel<4, false><<<grid, kAttnWarps * 32, 0, as_stream(stream)>>>(
            q, d, kc, vc, T_dev, max_ctx, scale, (__half*)out, nullptr, nullptr);
        return check_launch("pmpd_attention");
      case 256:
        attention_split_kernel<8, false><<<grid, kAttnWarps * 32, 0, as_stream(stream)>>>(
            q, d, kc, vc, T_dev, max_ctx, scale, (__half*)out, nullptr, nullptr);
        return check_launch("pmpd_attention");
      default:
        break;
    }
  }
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

int pmpd_attention_rope_batch(const float* qkv, int32_t ldqkv, int32_t m, int32_t d, int32_t d_head,
                              const float* cos_t, const float* sin_t, const int32_t* T_dev, int32_t max_ctx,
                              float scale, void* k_cache, void* v_cache, int64_t seq_stride, void* out,
                              void* stream) {
  if (d % d_head || d_head % 32 || d_head > 256) return fail(PMPD_ERR_CONFIG, "bad head geometry for the fused path");
  if (m < 1 || ldqkv < 3 * d) return fail(PMPD_ERR_CONFIG, "bad batch geometry (m >= 1, ldqkv >= 3d)");
  if ((reinterpret_cast<uintptr_t>(k_cache) & 15) || (reinterpret_cast<uintptr_t>(v_cache) & 15) || (seq_stride & 7))
    return fail(PMPD_ERR_INPUT, "KV caches must be 16-byte aligned");
  const dim3 grid((unsigned)(m * (d / d_head) * kSplit));
  auto kc = static_cast<__half*>(k_cache);
  auto vc = static_cast<__half*>(v_cache);
  auto o = static_cast<__half*>(out);
  const auto st = as_stream(stream);
  switch (d_head) {
    case 32:
      attention_split_kernel<1, true><<<grid, kAttnWarps * 32, 0, st>>>(qkv, d, kc, vc, T_dev, max_ctx, scale, o, cos_t,
                                                                         sin_t, ldqkv, seq_stride);
      break;
    case 64:
      attention_split_kernel<2, true><<<grid, kAttnWarps * 32, 0, st>>>(qkv, d, kc, vc, T_dev, max_ctx, scale, o, cos_t,
                                                                         sin_t, ldqkv, seq_stride);
      break;
    case 128:
      attention_split_kernel<4, true><<<grid, kAttnWarps * 32, 0, st>>>(qkv, d, kc, vc, T_dev, max_ctx, scale, o, cos_t,
                                                                         sin_t, ldqkv, seq_stride);
      break;
    case 256:
      attention_split_kernel<8, true><<<grid, kAttnWarps * 32, 0, st>>>(qkv, d, kc, vc, T_dev, max_ctx, scale, o, cos_t,
                                                                         sin_t, ldqkv, seq_stride);
      break;
    default:
      return fail(PMPD_ERR_CONFIG, "head dim %d not supported by the fused path", d_head);
  }
  return check_launch("pmpd_attention_rope_batch");
}

int pmpd_attention_rope(const float* qkv, int32_t d, int32_t d_head, const float* cos_t, const float* sin_t,
                        const int32_t* T_dev, int32_t max_ctx, float scale, void* k_cache, void* v_cache, void* out,
                        void* stream) {
  return pmpd_attention_rope_batch(qkv, 3 * d, 1, d, d_head, cos_t, sin_t, T_dev, max_ctx, scale, k_cache, v_cache, 0,
                                   out, stream);
}

int pmpd_silu_mul(const float* u, int32_t ldu, int32_t m, int32_t ff, void* out, int32_t ldo, void* stream) {
  if (m < 1 || ff < 1) return 0;
  if (m > 65535) return fail(PMPD_ERR_CONFIG, "silu_mul: at most 65535 rows, got %d", m);
  const int vec = (ldu % 4 == 0) && (ff % 4 == 0) && (ldo % 2 == 0) &&
                  (reinterpret_cast<uintptr_t>(u) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 3) == 0;
  const dim3 grid((unsigned)((ff + 4 * kBlock - 1) / (4 * kBlock)), (unsigned)m);
  silu_mul_kernel<<<grid, kBlock, 0, as_stream(stream)>>>(u, ldu, ff, m, (__half*)out, ldo, vec);
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

/*
 * pmpd_b200.h — C ABI of the B200-native PMPD quantized-linear hot path.
 *
 * The reference (arXiv 2410.13461 "PMPD", /root/reference/pkg/src/pmpd) is a
 * pure-Python/numpy package with no FFI of its own; its hot-path boundary is
 * a set of Python functions.  Each entry point below replaces one of them and
 * cites the reference interface it stands in for (file:line).  Python binds
 * this library with ctypes (paper_2410_13461_b200/_capi.py); INTEGRATION.md
 * shows the binding a reference maintainer would add.
 *
 * Conventions
 *  - All pointers named *_dev are device pointers; nothing here allocates
 *    device memory: callers own every buffer (torch tensors in the Python
 *    package).  Host-side metadata travels in plain C structs.
 *  - Every compute call is stream-ordered and asynchronous (no host sync), so
 *    it can be captured into a CUDA graph.  `stream` is a cudaStream_t passed
 *    as void* (0 = legacy default stream).
 *  - Return value: PMPD_OK (0) or an error class that mirrors the reference
 *    exception taxonomy (errors.py:8-25); pmpd_last_error() returns the
 *    message of the last failure on the calling thread.  The reference CLI maps
 *    Config/Input/Format errors to exit code 2 and ContractViolation to 3
 *    (cli.py:22-23).
 */
#ifndef PMPD_B200_H
#define PMPD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
#define PMPD_OK 0
#define PMPD_ERR_CONFIG 1   /* ConfigError: parameter outside its domain (errors.py:12) */
#define PMPD_ERR_INPUT 2    /* InputError: unusable user data (errors.py:16) */
#define PMPD_ERR_CONTRACT 3 /* ContractViolation (errors.py:24) */
#define PMPD_ERR_FORMAT 4   /* FormatError (errors.py:20) */
#define PMPD_ERR_CUDA 5     /* CUDA runtime failure (no reference counterpart) */

/* ------------------------------------------------------------------ layouts */
/* REF: the reference's own byte layout (quant.py:14-21): p_max MSB-first planes
 *      of ceil(rows*cols/8) bytes, row-major, LSB-first in bytes; scales are the
 *      reference mins[rows][groups] then deltas[rows][groups] (f32).
 *      Kernel orientation: y[r] = sum_c W[r][c] x[c] (n = rows, k = cols).
 * KN:  reference matrix stored (d_in, d_out) = (K, N) and applied as x @ W, as
 *      every tinylm matrix is (tinylm.py:119-127,341): groups run along N.
 * NK:  reference matrix stored (N, K) and applied as x @ W^T (BASELINE config
 *      1): groups run along K.
 * KN and NK are "tiled": 64x64 weight tiles, one contiguous region per bit
 * plane (reading precision p touches exactly planes 0..p-1, the reference's
 * memory-prefix property, quant.py:5-8), bits permuted inside each tile into
 * the tensor-core fragment order of the decode GEMV, plus a per-tile f32
 * scale block (and, for KN, a per-n-tile 1/max(step) used to scale the GEMV's
 * integer activation operand).  They require group_size % 64 == 0 and p_max <= 4. */
#define PMPD_LAYOUT_REF 0
#define PMPD_LAYOUT_KN 1
#define PMPD_LAYOUT_NK 2

#define PMPD_DTYPE_F32 0
#define PMPD_DTYPE_F16 1
#define PMPD_DTYPE_F64 2

/* One quantized matrix resident in HBM (QuantizedTensor, quant.py:116-139). */
typedef struct pmpd_qtensor {
  int32_t rows, cols;        /* reference shape */
  int32_t group_size, p_max; /* quant.py:157 arguments */
  int32_t layout;            /* PMPD_LAYOUT_* */
  int32_t n, k;              /* kernel orientation: y[n] = sum_k W[n,k] x[k] */
  int32_t n_tiles, k_tiles;  /* ceil(n/64), ceil(k/64) for tiled layouts */
  int32_t groups;            /* groups per reference row: ceil(cols/group_size) */
  int64_t plane_bytes;       /* bytes of ONE plane region */
  int64_t scale_bytes;       /* bytes of the scale region (after the planes) */
  int64_t aux_bytes;         /* KN: per n-tile 1/max(step) (after the scales); else 0 */
  int64_t total_bytes;       /* p_max * plane_bytes + scale_bytes + aux_bytes */
  void* data;                /* device base pointer, caller-owned */
} pmpd_qtensor;

/* Library/device identification; returns PMPD_OK. */
int pmpd_version(int32_t* major, int32_t* minor);
const char* pmpd_last_error(void);

/* Fill sizes/geometry of a quantized matrix (no allocation).
 * Replaces the shape bookkeeping of QuantizedTensor/BitPlaneStore
 * (quant.py:74-84,112-143).  CONFIG error for bad p_max/group_size/layout. */
int pmpd_qtensor_describe(int32_t rows, int32_t cols, int32_t group_size, int32_t p_max, int32_t layout,
                          pmpd_qtensor* out);

/* Bit-exact device quantizer: replaces quantize_tensor (quant.py:157-191).
 * w_dev: rows x cols weights (dtype PMPD_DTYPE_F32/F16/F64, row-major).
 * Outputs the REFERENCE representation: planes_dev [p_max][ceil(rows*cols/8)],
 * mins_dev/deltas_dev [rows][groups] f32.  codes_scratch_dev: rows*cols bytes.
 * Non-finite weights are reported through *nonfinite_dev (int32, set to 1);
 * the caller raises InputError after synchronizing. */
int pmpd_quantize(const void* w_dev, int32_t dtype, int32_t rows, int32_t cols, int32_t p_max, int32_t group_size,
                  uint8_t* codes_scratch_dev, uint8_t* planes_dev, float* mins_dev, float* deltas_dev,
                  int32_t* nonfinite_dev, void* stream);

/* Reference planes from integer codes (rows x cols u8, values < 2^p_max):
 * replaces BitPlaneStore.from_codes (quant.py:86-94). */
int pmpd_planes_from_codes(const uint8_t* codes_dev, int32_t rows, int32_t cols, int32_t p_max, uint8_t* planes_dev,
                           void* stream);

/* Pack the reference representation into t->layout inside t->data.
 * Replaces BitPlaneStore.from_codes (quant.py:86-94) as the producer of the
 * resident device copy. */
int pmpd_pack(const pmpd_qtensor* t, const uint8_t* ref_planes_dev, const float* mins_dev, const float* deltas_dev,
              void* stream);

/* Exact inverse of pmpd_pack (round-trip test of the packer). */
int pmpd_unpack(const pmpd_qtensor* t, uint8_t* ref_planes_dev, float* mins_dev, float* deltas_dev, void* stream);

/* Top-p codes of every weight, reference orientation (rows x cols u8):
 * replaces BitPlaneStore.prefix_codes / unpack_prefix (quant.py:96-105,194). */
int pmpd_prefix_codes(const pmpd_qtensor* t, int32_t p, uint8_t* codes_dev, void* stream);

/* Dequantize at precision p to f32, reference orientation (rows x cols).
 * Replaces dequantize (quant.py:199-215): w = fmaf(kidx, step, min) with
 * kidx = code (p == p_max) or code*2^m + 2^(m-1) (bucket centre, m = p_max-p);
 * equals float32(reference float64 result) bit for bit.  CONFIG error if p is
 * outside [1, p_max]. */
int pmpd_dequant(const pmpd_qtensor* t, int32_t p, float* out_dev, void* stream);

/* Rows `ids_dev[0..n)` of a REF-layout matrix dequantized at precision
 * *p_dev into out (f32, n x cols): the embedding gather
 * `weights("embed", p)[ids]` (tinylm.py:334). */
int pmpd_gather_rows(const pmpd_qtensor* t, const int32_t* ids_dev, int32_t n, const int32_t* p_dev, float* out_dev,
                     void* stream);

/* Bytes of scratch the GEMV needs for batch m (cross-CTA reduction). */
int pmpd_gemv_workspace_bytes(const pmpd_qtensor* t, int32_t m, int64_t* bytes);

/* Decode GEMV, batch 1..8: y[b][n] = alpha * sum_k W_p[n,k] x[b][k] (+ y if accumulate).
 * Replaces `h @ model.weights(name, p)` at every linear call site of the
 * decode loop (tinylm.py:201-231 + 341-368).  The active precision is read
 * from device memory (*p_dev) so a precision switch needs no host sync and no
 * weight reload; only planes 0..p-1 are read.  x: f16 [m][ldx]; y: f32 or f16
 * [m][ldy].  workspace_dev must be zero-initialised once (its counters are
 * self-resetting).  Launched with programmatic dependent launch: weights are
 * prefetched before the kernel waits on its predecessor's activations. */
int pmpd_gemv(const pmpd_qtensor* t, const void* x_dev, int32_t ldx, int32_t m, const int32_t* p_dev, void* y_dev,
              int32_t y_dtype, int32_t ldy, float alpha, int32_t accumulate, void* workspace_dev,
              int64_t workspace_bytes, void* stream);

/* Decode GEMV with its producer op fused into the activation staging (batch 1..8, staged path:
 * K <= 12288 at m = 1, m*K <= 32768 otherwise; CONFIG error outside it, callers then run the
 * two ops separately):
 *   PMPD_GEMV_IN_RMSNORM: x = f16(xf * rsqrt(mean(xf^2) + eps) * gain)   (tinylm.py:293-295,
 *                         the RMSNorm before q|k|v and before gate|up, 337/345)
 *   PMPD_GEMV_IN_SWIGLU:  x = f16(silu(xf[k]) * xf[k + u_off])            (tinylm.py:298,362-364,
 *                         the SwiGLU before the down projection)
 * xf: f32 [m][ldxf]; everything else as pmpd_gemv. */
#define PMPD_GEMV_IN_RMSNORM 1
#define PMPD_GEMV_IN_SWIGLU 2
int pmpd_gemv_fused(const pmpd_qtensor* t, int32_t in_mode, const float* xf_dev, int32_t ldxf, int32_t m,
                    const float* gain_dev, float eps, int32_t u_off, const int32_t* p_dev, void* y_dev,
                    int32_t y_dtype, int32_t ldy, float alpha, int32_t accumulate, void* workspace_dev,
                    int64_t workspace_bytes, void* stream);

/* Prefill GEMM on sm_100a tensor cores (tcgen05, TMEM accumulators): the
 * prompt-length linear layers of prefill (tinylm.py:377-388 -> 334-368).
 * y[m][n] = alpha * sum_k x[m][k] W_p[n][k] (+ y if accumulate) for m >= 1 rows;
 * each CTA dequantizes its weight tiles bit-exactly (f32 min + k*step, quant.py:199-215)
 * to f16 in shared memory once and runs them against 128 rows of x.  KN tiles,
 * p_max 4, K a multiple of 64; x: f16 [m][ldx] (16-byte aligned rows); y: f32 or
 * f16 [m][ldy].  *p_dev is the precision (1..p_max); an out-of-range value sets
 * *status_dev (optional) to PMPD_ERR_CONTRACT and is clamped. */
int pmpd_gemm(const pmpd_qtensor* t, const void* x_dev, int32_t ldx, int32_t m, const int32_t* p_dev, void* y_dev,
              int32_t y_dtype, int32_t ldy, float alpha, int32_t accumulate, int32_t* status_dev, void* stream);

/* Per-token precision hook: replaces PrecisionSchedule.precision_at
 * (schedule.py:93-99) as called by generate (tinylm.py:512,518).
 * sched_dev: int32 [2*n_prec] = {p_0, st_0, p_1, st_1, ...} (any order; entries
 * with p <= 0 are unused, so a fixed-capacity table can be rewritten in place
 * without re-capturing a CUDA graph);
 * step_dev: int32 decode-step counter.  Writes the lowest precision whose
 * switch point is <= *step_dev to *p_out_dev, then (if advance) increments
 * *step_dev.  Entirely on device: no host sync inside a captured decode step. */
int pmpd_sched_step(const int32_t* sched_dev, int32_t n_prec, int32_t* step_dev, int32_t* p_out_dev, int32_t advance,
                    void* stream);

/* ------------------------------------------------------------- decode engine
 * All quantized linear layers of one batch-1 decode token in ONE cooperative
 * persistent kernel (replaces the per-layer h @ weights(name, p) calls of a
 * reference decode step, tinylm.py:341-368).  A program is a device array of
 * opaque op records (pmpd_engine_op_bytes() each) built with
 * pmpd_engine_make_op + pmpd_engine_op_set_bounds + pmpd_engine_op_set_counted;
 * op i reads the f16 vector in_alpha * (output of op src)[src_col ...] (act 0)
 * or silu(g)*u (act 1), or x_in for src = -1.  Split-K partials are added into
 * counted fixed-point words (see pmpd_engine_op_set_counted): deterministic,
 * and complete when their contributor count is reached, so ops follow each other
 * without a grid barrier.  The last op's output lands in y_out (f32) scaled by
 * y_alpha.  bar_dev: 3 + 2 * n_ops zero-initialised uint32 (epoch and counters,
 * kept across launches).  Weights are streamed at the precision *p_dev (planes
 * 0..p-1 only).  part_dev / max_slots of pmpd_engine_make_op are unused (ABI). */
int pmpd_engine_op_bytes(void);
int pmpd_engine_grid(void);
int pmpd_engine_max_slots(const pmpd_qtensor* t);
/* Contributing CTAs per n-group of t's output under the engine grid (host array, n_tiles bytes). */
int pmpd_engine_nslots(const pmpd_qtensor* t, uint8_t* out_host);
int pmpd_engine_make_op(const pmpd_qtensor* t, int32_t src, int32_t src_col, int32_t act, int32_t act_off,
                        float in_alpha, float* part_dev, int32_t max_slots, const uint8_t* nslots_dev,
                        void* op_host);
/* Decoder-step ops (a whole batch-1 decode step in one engine launch; tinylm.py:334-368):
 *   pmpd_engine_op_set_io: after pmpd_engine_make_op, switch the op's input to
 *     in_mode 2 = RMSNorm(residual stream) * gain over the whole row (tinylm.py:293-295,
 *     337/345/349) or in_mode 3 = the combined records of the attention op `src`; keep_out = 1
 *     makes the op a residual op (its output is ADDED into the residual stream, x += ctx @ Wo /
 *     x += a @ W_down, tinylm.py:359/364), scaled by out_alpha.  resid_dev is unused (the stream
 *     is an argument of pmpd_engine_run_decoder).
 *   pmpd_engine_make_attn_op: attention over one layer's f16 KV cache for the new token: q|k|v =
 *     the output of op `src`; RoPE at position T = *T_dev (cos/sin [max_ctx][d_head/2]);
 *     k, v appended to row T; records_dev = u64 [3][pmpd_engine_attn_records()].
 *     d_head in {32, 64, 128, 256}. */
int pmpd_engine_op_set_io(void* op_host, int32_t in_mode, const float* resid_dev, const float* gain_dev, float eps,
                          int32_t keep_out, float out_alpha);
int pmpd_engine_make_attn_op(int32_t src, int32_t n_heads, int32_t d_head, void* k_cache_dev, void* v_cache_dev,
                             const float* cos_dev, const float* sin_dev, const int32_t* T_dev, int32_t max_ctx,
                             float scale, void* records_dev, void* op_host);
int pmpd_engine_attn_records(int32_t n_heads, int32_t d_head);
/* Cost-balanced CTA tile ranges for one op (bounds_host: pmpd_engine_grid() + 1 ints): the ranges
 * minimise the largest per-CTA cost of stage calls and n-group flushes instead of splitting the tiles
 * evenly; attach the uploaded array with pmpd_engine_op_set_bounds (null = even split). */
int pmpd_engine_partition(const pmpd_qtensor* t, int32_t* bounds_host);
/* The same over G CTAs (a rank's share of the grid in pmpd_engine_run_ranks). */
int pmpd_engine_partition_g(const pmpd_qtensor* t, int32_t G, int32_t* bounds_host);
/* The same with a per-CTA budget reduction delta_host[G] (in half tile-times, >= 0): CTAs measured
 * slower than the rest (later input, slower tiles: a property of their SM's place in the chip)
 * get proportionally less work (calibrated by engine.calibrate_deltas from a traced token). */
int pmpd_engine_partition_w(const pmpd_qtensor* t, int32_t G, const int32_t* delta_host, int32_t* bounds_host);
int pmpd_engine_op_set_bounds(void* op_host, const int32_t* bounds_dev);
/* Counted accumulation (linear-stack programs run by pmpd_engine_run): the op's output is
 * acc_dev = u64 [3][n_tiles * 64] zero-initialised words, each holding [63:54] the number of CTAs
 * that added into it and [53:0] the sum of their partials as 2^-24 fixed point (offset binary),
 * so split-K sums are bit-reproducible and self-validating; nslots_dev[n_tiles] = contributors
 * per n-group under the op's bounds, n_contrib = CTAs with a nonempty range.  bar_dev of the run
 * then holds 3 + n_ops u32 (tickets, done, launch epoch, per-op hint counters), zeroed once. */
int pmpd_engine_op_set_counted(void* op_host, void* acc_dev, const uint8_t* nslots_dev, int32_t n_contrib);
/* Sub-ops: restrict an op (before set_io / set_counted) to n-groups [ng0, ng1) and k-tiles
 * [kt0, kt1) of its tensor.  The sub-op reads input elements kt0*64.. of its source and adds into
 * the tensor's whole output vector (set_counted with the vector's base; every sub-op of one tensor
 * passes the same acc_dev / nslots_dev, the counts summed over the sub-ops' partitions), so a row-
 * parallel op can run as k-slices whose CTAs depend only on the source n-groups of their slice.
 * set_share: zero_output = 0 for all but one sub-op of a shared output (that one zeroes the idle
 * set of the whole vector). */
int pmpd_engine_op_set_slice(void* op_host, int32_t ng0, int32_t ng1, int32_t kt0, int32_t kt1);
int pmpd_engine_op_set_share(void* op_host, int32_t zero_output);
/* Final step of building an op table (host copy, before it is uploaded): copies each op's source
 * output (counted vector, counts, scope) into the op record.  Required after set_counted /
 * set_peers of every op. */
int pmpd_engine_link(void* ops_host, int32_t n_ops);
/* Decoder programs (pmpd_engine_run_decoder): every linear op is counted (pmpd_engine_op_set_counted);
 * the o / down ops (keep_out) add into ONE counted residual stream resid_dev = u64 [3][resid_len]
 * (resid_len = d rounded up to 64, zero-initialised), into which the launch first adds x0_dev (f32
 * [d_real], the embedding row written before the launch).  An RMSNorm op reads the stream when each
 * word's contribution count reaches cum_dev[n-group] (u16, static: 1 + the contributors of every
 * residual op before it); a residual op passes rwait = the index of the RMSNorm op whose readers
 * must have read the stream before it adds (-1: none).  Attention records are single-writer words,
 * records_dev = u64 [3][pmpd_engine_attn_records()].  bar_dev holds 3 + 2 * n_ops u32. */
int pmpd_engine_op_set_residual(void* op_host, const uint16_t* cum_dev, int32_t rwait);
int pmpd_engine_run_decoder(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const float* x0_dev,
                            void* resid_dev, int64_t resid_len, int32_t d_real, float* y_out_dev, float y_alpha,
                            uint32_t* bar_dev, int32_t* status_dev, int64_t* trace_dev, void* stream);

/* Tensor-parallel linear stack, all ranks emulated in ONE launch (one GPU): ops_dev holds n_ranks
 * op tables of n_ops records (rank r = its column / row shards, partitioned with
 * pmpd_engine_partition_g over pmpd_engine_grid() / n_ranks CTAs); the grid is split into n_ranks
 * groups, group r runs table r and writes y_out + r * y_stride.  A row-parallel op's counted output
 * is one vector shared by every rank's op record, with contributor counts summed over the ranks:
 * the cross-rank all-reduce is the counted addition itself (no collective call). */
/* Row-parallel op of a tensor-parallel program: add every partial into each of the n_peers copies
 * of the op's output (this rank's own copy among them: the copies are the ranks' symmetric
 * buffers, u64 [3][n_tiles * 64] each); sys_scope = 1 when the copies live on other GPUs
 * (system-scope additions and polls over NVLink). */
int pmpd_engine_op_set_peers(void* op_host, const void* const* peers_host, int32_t n_peers, int32_t sys_scope);
int pmpd_engine_run_ranks(const void* ops_dev, int32_t n_ops, int32_t n_ranks, const int32_t* p_dev,
                          const void* x_in_dev, float* y_out_dev, int32_t y_stride, float y_alpha, uint32_t* bar_dev,
                          int32_t* status_dev, void* stream);
int pmpd_engine_run(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const void* x_in_dev, float* y_out_dev,
                    float y_alpha, uint32_t* bar_dev, int32_t* status_dev, void* stream);
/* Same, recording a per-CTA per-op timeline (globaltimer ns):
 * {input ready, input staged, tiles done, op published, warp-0 cycles in tiles, tile calls, loop cycles, 0}
 * (trace_dev is [grid][n_ops][8]). */
int pmpd_engine_run_traced(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const void* x_in_dev,
                           float* y_out_dev, float y_alpha, uint32_t* bar_dev, int32_t* status_dev, int64_t* trace_dev,
                           void* stream);

/* ------------------------------------------------------------- decoder glue
 * The non-linear parts of one forward step (tinylm.py:293-368); residual
 * stream f32, GEMV inputs f16, KV cache f16 [max_ctx][d] per layer holding
 * post-RoPE K and V rows (KVCache, tinylm.py:272-286).  *T_dev is the number
 * of cached tokens before the step, read on device (graph-replayable). */

/* out (f16, ldo) = x / sqrt(mean(x^2) + eps) * gain, per row (_rmsnorm, tinylm.py:293-295). */
int pmpd_rmsnorm(const float* x_dev, int32_t ldx, const float* gain_dev, int32_t m, int32_t d, float eps, void* out_dev,
                 int32_t ldo, void* stream);

/* Rotate-half RoPE of q|k (tinylm.py:308-319,344-345) for m tokens at positions
 * *T_dev + i; rotated q -> q_out (f32 [m][d]); rotated k and v -> cache rows
 * (tinylm.py:346-347).  cos/sin: f32 [max_ctx][d_head/2] from float64 tables. */
int pmpd_rope_kv(const float* qkv_dev, int32_t ldq, int32_t m, int32_t d, int32_t d_head, const float* cos_dev,
                 const float* sin_dev, const int32_t* T_dev, int32_t max_ctx, float* q_out_dev, void* k_cache_dev,
                 void* v_cache_dev, void* stream);

/* Causal softmax attention of m queries over cache rows 0..T+i (tinylm.py:349-358) -> f16 [m][d]. */
int pmpd_attention(const float* q_dev, int32_t m, int32_t d, int32_t d_head, const void* k_cache_dev,
                   const void* v_cache_dev, const int32_t* T_dev, int32_t max_ctx, float scale, void* out_dev,
                   void* stream);

/* Decode step (one query) with RoPE and the KV append fused into the split-context attention:
 * q|k|v of the new token (f32 row: q at 0, k at d, v at 2d) -> rotate q and k at position
 * T = *T_dev (tinylm.py:308-319,344-347), write k and v into cache row T (f16, skipped when
 * T >= max_ctx), attend over rows 0..T (tinylm.py:349-358) -> out f16 [d].  Equals
 * pmpd_rope_kv followed by pmpd_attention for m = 1.  d_head in {32, 64, 128, 256}. */
int pmpd_attention_rope(const float* qkv_dev, int32_t d, int32_t d_head, const float* cos_dev, const float* sin_dev,
                        const int32_t* T_dev, int32_t max_ctx, float scale, void* k_cache_dev, void* v_cache_dev,
                        void* out_dev, void* stream);

/* Batched decode: m independent sequences, one new token each.  Row i of qkv_dev (stride ldqkv
 * >= 3d) is sequence i's q|k|v; its cache is k_cache_dev / v_cache_dev + i * seq_stride halfs
 * ([max_ctx][d] f16 rows) with length T_dev[i]; same math per sequence as pmpd_attention_rope.
 * Output row i (stride d).  Replaces a per-sequence loop of pmpd_attention_rope calls. */
int pmpd_attention_rope_batch(const float* qkv_dev, int32_t ldqkv, int32_t m, int32_t d, int32_t d_head,
                              const float* cos_dev, const float* sin_dev, const int32_t* T_dev, int32_t max_ctx,
                              float scale, void* k_cache_dev, void* v_cache_dev, int64_t seq_stride, void* out_dev,
                              void* stream);

/* out (f16) = silu(u[:, :ff]) * u[:, ff:] (tinylm.py:362-364). */
int pmpd_silu_mul(const float* u_dev, int32_t ldu, int32_t m, int32_t ff, void* out_dev, int32_t ldo, void* stream);

/* Greedy sample: argmax per row, lowest index on ties (sample, tinylm.py:422-429);
 * sets *bad_dev = 1 if a logit is non-finite (InputError in the reference). */
int pmpd_argmax(const float* logits_dev, int32_t ld, int32_t m, int32_t vocab, int32_t* out_dev, int32_t* bad_dev,
                void* stream);

/* *p += v on device (cache-length and step counters). */
int pmpd_add_i32(int32_t* p_dev, int32_t v, void* stream);

/* dst[*idx_dev][0..n) = src[0..n) if *idx_dev < capacity (per-step logits history). */
int pmpd_store_row(const float* src_dev, float* dst_dev, const int32_t* idx_dev, int32_t n, int32_t capacity,
                   void* stream);

/* Device bookkeeping of one generated token: tokens[*n] = *cur; *n += 1; *T += 1 (if T). */
int pmpd_push_token(const int32_t* cur_dev, int32_t* tokens_dev, int32_t* n_dev, int32_t* T_dev, int32_t capacity,
                    void* stream);

/* Learned switch predictor on device (learnsched.py:118-125,151-160):
 * attention-pool cache rows 0..T-1 of the feature block with query q, ReLU MLP,
 * argmax (lowest on ties) -> grid point; writes the two-phase schedule
 * {p_high: 0, p_low: grid[cls]} into the fixed-capacity table sched_dev
 * (int32[16], the pmpd_sched_step format).  dbg_logits (optional, f32[ncls]). */
int pmpd_learned_predict(const void* k_dev, const void* v_dev, int32_t ldkv, const int32_t* T_dev, int32_t max_T,
                         int32_t dk, int32_t dv, int32_t hidden, int32_t ncls, const float* q_dev, const float* w1_dev,
                         const float* b1_dev, const float* w2_dev, const float* b2_dev, const int32_t* grid_dev,
                         int32_t p_high, int32_t p_low, int32_t* sched_dev, float* dbg_logits_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PMPD_B200_H */

// Packed bit-plane layout of the tiled formats (PMPD_LAYOUT_KN / _NK).
//
// A 64x64 tile (n_l, k_l) is consumed by one warp as 4 m-tiles (t = n_l/16)
// x 4 k-tiles (w = k_l/16) of the m16n8k16 tensor-core instruction, with the
// weights in the A operand (swap-AB decode GEMV).  Lane L = 4*gq + tig of the
// warp reads, per bit plane, one 16-byte chunk = 4 u32 words (w = 0..3).  Word
// w of plane j holds bit b_j = p_max-1-j of 32 codes: (t, s) for t = 0..3
// m-tiles and s = 0..7 "nibble slots", at bit position (4s + t + b_j) mod 32.
//
// Consumer decode (gemv.cu): OR-ing the p masked plane words of one (w, t)
// gives a word whose nibble slot s holds the 4-bit bucket index of weight
// (t, s) shifted left by t bits; masking two slot pairs per half2 and OR-ing
// an fp16 exponent turns them straight into fp16 values 2^(10-t)+k (slots
// 0,4 / 2,6) and 2^(6-t)+k (slots 1,5 / 3,7) for the A fragment registers
// a0..a3, with no shifts beyond one 8-bit rotate per word.  The per-row
// offsets are removed exactly after the MMA.
//
// The slot -> (row, k) map differs per layout (see nk_/kn_tile_coord below):
// NK tiles feed fp16 A fragments of mma.m16n8k16 (per-row f32 scales need
// f32 accumulators per tile); KN tiles feed u8 A fragments of mma.m16n8k32
// whose bytes are the bucket indices themselves (int32 accumulation).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define PMPD_HD __host__ __device__ __forceinline__
#else
#define PMPD_HD inline
#endif

namespace pmpd {

struct TileCoord {
  int lane, w, t, s;
};

// ---- NK tiles: fragment order of mma.m16n8k16 (fp16 A, HMMA decode path) ----
// slot s: row = gq + 8*(s&1), k = 16w + 2*tig + 8*((s>>1)&1) + (s>>2)
PMPD_HD TileCoord nk_tile_coord(int n_l, int k_l) {
  TileCoord c;
  c.t = n_l >> 4;
  const int r = n_l & 15;
  const int gq = r & 7, h = r >> 3;
  c.w = k_l >> 4;
  const int kk = k_l & 15;
  const int tig = (kk & 7) >> 1, e = kk & 1, hi8 = kk >> 3;
  c.s = h + 2 * hi8 + 4 * e;
  c.lane = gq * 4 + tig;
  return c;
}
PMPD_HD void nk_tile_inverse(int lane, int w, int t, int s, int* n_l, int* k_l) {
  const int gq = lane >> 2, tig = lane & 3;
  *n_l = 16 * t + gq + 8 * (s & 1);
  *k_l = 16 * w + 2 * tig + 8 * ((s >> 1) & 1) + (s >> 2);
}

// ---- KN tiles: fragment order of mma.m16n8k32 (u8 A, IMMA decode path) ----
// A fragment (m-tile t, 32-k chunk c): a0/a1 = even/odd slots of word w = 2c,
// a2/a3 = even/odd slots of word w = 2c+1; a register holds 4 consecutive k.
// slot s: row = gq + 8*(s&1), k = 32*(w>>1) + 16*(w&1) + 4*tig + (s>>1)
PMPD_HD TileCoord kn_tile_coord(int n_l, int k_l) {
  TileCoord c;
  c.t = n_l >> 4;
  const int r = n_l & 15;
  const int gq = r & 7, h = r >> 3;
  c.w = ((k_l >> 5) << 1) | ((k_l >> 4) & 1);
  const int kk = k_l & 15;
  const int tig = kk >> 2, j = kk & 3;
  c.s = h + 2 * j;
  c.lane = gq * 4 + tig;
  return c;
}
PMPD_HD void kn_tile_inverse(int lane, int w, int t, int s, int* n_l, int* k_l) {
  const int gq = lane >> 2, tig = lane & 3;
  *n_l = 16 * t + gq + 8 * (s & 1);
  *k_l = 32 * (w >> 1) + 16 * (w & 1) + 4 * tig + (s >> 1);
}

PMPD_HD TileCoord tile_coord(bool kn, int n_l, int k_l) { return kn ? kn_tile_coord(n_l, k_l) : nk_tile_coord(n_l, k_l); }
PMPD_HD void tile_inverse(bool kn, int lane, int w, int t, int s, int* n_l, int* k_l) {
  if (kn)
    kn_tile_inverse(lane, w, t, s, n_l, k_l);
  else
    nk_tile_inverse(lane, w, t, s, n_l, k_l);
}

// bit position inside the plane word: nibble slot s of m-tile t, code bit b_j
PMPD_HD int tile_bitpos(int t, int s, int bj) { return (4 * s + t + bj) & 31; }

// u32 word index of (lane, w) inside a tile's 512-byte plane chunk
PMPD_HD int tile_word(int lane, int w) { return lane * 4 + w; }

// Order of the 64 per-row scales inside an NK tile scale block: lane group gq
// reads its 8 rows (t = 0..3, h = 0..1) as two 16-byte vectors.
PMPD_HD int nk_scale_slot(int n_l) {
  const int t = n_l >> 4, r = n_l & 15, gq = r & 7, h = r >> 3;
  return gq * 8 + t * 2 + h;
}

}  // namespace pmpd

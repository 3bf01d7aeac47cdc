// Bit-plane -> tensor-core fragment decode shared by the decode GEMV (gemv.cu)
// and the persistent decode engine (engine.cu).  See layout.cuh for the
// packed tile layout these functions assume.
#pragma once
#include "pmpd_common.cuh"

namespace pmpd {

// ---------------------------------------------------------------- decode core
// Merge planes 0..P-1 of word (w, t) into a nibble word.  Plane j's bits for
// m-tile t sit at rotl(0x11111111 << b_j, t); bit-selecting keeps each
// plane's own positions (positions of unread planes hold garbage that the
// fragment conversion masks off).  One LOP3 per extra plane.
template <int PMAX, int P, int T>
PMPD_DEV uint32_t merge_planes(const uint32_t (&pw)[4]) {
  uint32_t acc = pw[0];
#pragma unroll
  for (int j = 1; j < P; ++j) {
    // positions already owned by planes 0..j-1, rotated by T (a compile-time immediate)
    const uint32_t have = (0x11111111u * (((1u << j) - 1) << (PMAX - j))) ;
    const uint32_t sel = (have << T) | (T ? (have >> (32 - T)) : 0u);
    acc = lop3_select(acc, pw[j], sel);
  }
  return acc;
}

// Decode position of the low slot pair for m-tile T: the nibble word is read
// rotated by R1 = T - Q0 so that slots (0,4)/(1,5) sit at mantissa bits
// Q0..Q0+3 / Q0+4..Q0+7 (both <= bit 9) and, after a further 8-bit rotate,
// slots (2,6)/(3,7) likewise.
template <int T>
struct FragPos {
  static constexpr int Q0 = T < 2 ? T : 2;
  static constexpr int R1 = T - Q0;
};

// fp16 A fragment from one nibble word of m-tile T (see layout.cuh).  OR-ing
// the exponent of 2^(10-q) onto a code at mantissa bits q..q+3 makes the half
// exactly 2^(10-q) + k (k = bucket index, exact in fp16).
template <int PMAX, int P, int T>
PMPD_DEV void nibble_to_frag(uint32_t u, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
  constexpr int Q0 = FragPos<T>::Q0, R1 = FragPos<T>::R1;
  // nibble bits that come from loaded planes, and the constant bucket-centre bit
  constexpr uint32_t kLoaded = ((1u << PMAX) - 1) & ~((1u << (PMAX - P)) - 1);
  constexpr uint32_t kConst = (P < PMAX) ? (1u << (PMAX - P - 1)) : 0u;
  constexpr uint32_t m0 = (kLoaded * 0x00010001u) << Q0;
  constexpr uint32_t m4 = (kLoaded * 0x00010001u) << (Q0 + 4);
  constexpr uint32_t g0 = (((uint32_t)(25 - Q0) << 10) | (kConst << Q0)) * 0x00010001u;
  constexpr uint32_t g4 = (((uint32_t)(21 - Q0) << 10) | (kConst << (Q0 + 4))) * 0x00010001u;
  const uint32_t ua = R1 ? rotr32(u, R1) : u;
  const uint32_t ub = rotr32(u, R1 + 8);
  a0 = lop3_and_or(ua, m0, g0);
  a1 = lop3_and_or(ua, m4, g4);
  a2 = lop3_and_or(ub, m0, g0);
  a3 = lop3_and_or(ub, m4, g4);
}

// fp16 value offset carried by each A row after the MMA: 2^(10-Q0) for rows
// gq (a0/a2), 2^(6-Q0) for rows gq+8 (a1/a3).
PMPD_DEV float row_offset(int t, int h) {
  const int q0 = t < 2 ? t : 2;
  return (float)(1024 >> (q0 + 4 * h));
}

// KN (IMMA) decode: u8 A fragment halves from one nibble word of m-tile T.
// Even slots (row gq) land in bytes 0..3 of `lo`, odd slots (row gq+8) in
// `hi`; every byte is bucket_index << T (<= 120), so the MMA result of m-tile
// T is 2^T times the true dot product (removed exactly at the flush).
template <int PMAX, int P, int T>
PMPD_DEV void nibble_to_u8(uint32_t u, uint32_t& lo, uint32_t& hi) {
  constexpr uint32_t kLoaded = ((1u << PMAX) - 1) & ~((1u << (PMAX - P)) - 1);
  constexpr uint32_t kConst = (P < PMAX) ? (1u << (PMAX - P - 1)) : 0u;
  constexpr uint32_t m = (kLoaded * 0x01010101u) << T;
  constexpr uint32_t cb = (kConst * 0x01010101u) << T;
  lo = lop3_and_or(u, m, cb);
  hi = lop3_and_or(rotr32(u, 4), m, cb);
}

}  // namespace pmpd

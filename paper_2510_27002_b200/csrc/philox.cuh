// Device Philox4x64-10 bit-exact with numpy's Philox bit generator
// (numpy/random/src/philox/philox.h), the generator deskworld.rng.stream wraps
// (rng.py:38-44).  Draw i of a state (counter c, buffer_pos p, buffer w) is
//   i <  4-p : w[p+i]
//   i >= 4-p : word (i-(4-p))%4 of Philox(c + 1 + (i-(4-p))/4, key)
// and next_double = (u64 >> 11) * 2^-53.
#pragma once
#include <stdint.h>

namespace jz {

struct PhiloxState {
  uint64_t ctr[4];
  uint64_t key[2];
  uint64_t buf[4];
  int pos;
};

__device__ __forceinline__ void philox4x64_10(const uint64_t (&c_in)[4], uint64_t k0, uint64_t k1,
                                              uint64_t (&out)[4]) {
  uint64_t c0 = c_in[0], c1 = c_in[1], c2 = c_in[2], c3 = c_in[3];
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
    const uint64_t lo1 = 0xCA5A826395121157ull * c2, hi1 = __umul64hi(0xCA5A826395121157ull, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// 256-bit counter + small increment
__device__ __forceinline__ void ctr_add(const uint64_t (&c)[4], uint64_t inc, uint64_t (&o)[4]) {
  o[0] = c[0] + inc;
  uint64_t carry = o[0] < c[0];
  o[1] = c[1] + carry; carry = carry && (o[1] == 0);
  o[2] = c[2] + carry; carry = carry && (o[2] == 0);
  o[3] = c[3] + carry;
}

// block index relative to the state (block j covers draws avail + 4j .. avail + 4j + 3)
__device__ __forceinline__ void philox_block(const PhiloxState& s, uint64_t j, uint64_t (&out)[4]) {
  uint64_t c[4];
  ctr_add(s.ctr, j + 1, c);
  philox4x64_10(c, s.key[0], s.key[1], out);
}

__device__ __forceinline__ uint64_t philox_word(const PhiloxState& s, uint64_t i) {
  const uint64_t avail = 4 - s.pos;
  if (i < avail) return s.buf[s.pos + i];
  const uint64_t k = i - avail;
  uint64_t w[4];
  philox_block(s, k >> 2, w);
  return w[k & 3];
}

__device__ __forceinline__ double u64_to_double(uint64_t w) {
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

}  // namespace jz

// CPython's random.Random on the device (Modules/_randommodule.c, Lib/random.py), bit for bit:
// MT19937 seeded by init_by_array with the 32-bit words of abs(seed), genrand_uint32, random()
// (two draws, 53 bits), getrandbits(k <= 32) and _randbelow_with_getrandbits.
//
// The init_genrand(19650218) table that init_by_array starts from does not depend on the seed,
// so it is a compile-time constant (kMtInit) read through the constant cache: every lane of a
// warp reads the same word at the same iteration, which is the constant cache's broadcast case.
#pragma once

#include <cstdint>

namespace cs {
namespace {

struct MtInitTable {
  uint32_t v[624];
  constexpr MtInitTable() : v() {
    v[0] = 19650218u;
    for (int i = 1; i < 624; ++i) v[i] = 1812433253u * (v[i - 1] ^ (v[i - 1] >> 30)) + (uint32_t)i;
  }
};

__constant__ MtInitTable kMtInit = MtInitTable();

struct Mt {
  uint32_t mt[624];
  int mti;
};

// init_by_array(key, key_len) (Modules/_randommodule.c)
__device__ __forceinline__ void mt_seed(Mt& s, const uint32_t* key, int key_len) {
  uint32_t prev = kMtInit.v[0];
  s.mt[0] = prev;
  int i = 1, j = 0;
  bool wrapped = false;  // before the first wrap every position still holds its kMtInit value
  // first sweep: fold the key into the init_genrand table (positions 1..623, then 1 again)
  for (int k = 624 > key_len ? 624 : key_len; k; --k) {
    const uint32_t cur = wrapped ? s.mt[i] : kMtInit.v[i];
    const uint32_t v = (cur ^ ((prev ^ (prev >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
    s.mt[i] = v;
    prev = v;
    ++i, ++j;
    if (i >= 624) s.mt[0] = v, i = 1, wrapped = true;
    if (j >= key_len) j = 0;
  }
  prev = s.mt[i - 1];
  for (int k = 623; k; --k) {
    const uint32_t v = (s.mt[i] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)i;
    s.mt[i] = v;
    prev = v;
    ++i;
    if (i >= 624) s.mt[0] = v, i = 1;
  }
  s.mt[0] = 0x80000000u;
  s.mti = 624;
}

__device__ __forceinline__ uint32_t mt_temper(uint32_t y) {
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= (y >> 18);
  return y;
}

__device__ __forceinline__ uint32_t mt_twist1(uint32_t a, uint32_t b, uint32_t c) {
  const uint32_t y = (a & 0x80000000u) | (b & 0x7fffffffu);
  return c ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
}

// genrand_uint32
__device__ __forceinline__ uint32_t mt_next(Mt& s) {
  if (s.mti >= 624) {
    for (int kk = 0; kk < 624; ++kk) {
      const int k1 = kk + 1 == 624 ? 0 : kk + 1;
      const int k397 = kk + 397 >= 624 ? kk + 397 - 624 : kk + 397;
      s.mt[kk] = mt_twist1(s.mt[kk], s.mt[k1], s.mt[k397]);
    }
    s.mti = 0;
  }
  return mt_temper(s.mt[s.mti++]);
}

// random() = (a * 2^26 + b) / 2^53
__device__ __forceinline__ double mt_random(Mt& s) {
  const uint32_t a = mt_next(s) >> 5, b = mt_next(s) >> 6;
  return __dmul_rn(__dadd_rn(__dmul_rn((double)a, 67108864.0), (double)b), 1.0 / 9007199254740992.0);
}

// The first 227 outputs after seeding need only the untwisted state (output kk < 227 reads
// mt[kk], mt[kk+1], mt[kk+397], none of which the twist has rewritten yet), so a short draw
// sequence skips the 624-word twist; the full twist runs only if output 227 is ever needed.
struct MtLazy {
  Mt s;
  int n;  // outputs drawn since seeding
};

__device__ __forceinline__ void mt_lazy_seed(MtLazy& r, const uint32_t* key, int key_len) {
  mt_seed(r.s, key, key_len);
  r.n = 0;
}

__device__ __forceinline__ uint32_t mt_lazy_next(MtLazy& r) {
  if (r.n < 227) {
    const int kk = r.n++;
    return mt_temper(mt_twist1(r.s.mt[kk], r.s.mt[kk + 1], r.s.mt[kk + 397]));
  }
  if (r.n == 227) {  // catch up: the standard full twist, then continue at output 227
    r.s.mti = 624;
    (void)mt_next(r.s);
    r.s.mti = 227;
  }
  ++r.n;
  return mt_next(r.s);
}

// Random.getrandbits(k) for 1 <= k <= 32, then _randbelow_with_getrandbits(n), n >= 1
__device__ __forceinline__ uint32_t mt_randbelow(MtLazy& r, uint32_t n) {
  const int k = 32 - __clz(n);
  uint32_t v = mt_lazy_next(r) >> (32 - k);
  while (v >= n) v = mt_lazy_next(r) >> (32 - k);
  return v;
}

}  // namespace
}  // namespace cs

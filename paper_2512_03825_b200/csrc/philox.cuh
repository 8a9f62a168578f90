// philox.cuh -- counter-based generators used on the device.
//
//  * Philox4x64-10, word 0 only: the reference's draw (isingpt rng.py:40-61),
//    counter (pos, 0, stream, 0), key (seed, stream).  Used by the exact
//    (reference-chain) kernels, the exact-count init and the swap decisions
//    (rng.py:99-116, kernels.py:130).
//  * Philox4x32-10 (Random123 constants): the checkerboard kernels' acceptance
//    stream; all four output words are consumed.
#pragma once
#include <cstdint>

namespace ptmh {

// ---------------------------------------------------------- Philox4x64-10 --
constexpr uint64_t kPh64M0 = 0xD2E7470EE14C6C93ULL;  // rng.py:18
constexpr uint64_t kPh64M1 = 0xCA5A826395121157ULL;  // rng.py:19
constexpr uint64_t kPh64W0 = 0x9E3779B97F4A7C15ULL;  // rng.py:20
constexpr uint64_t kPh64W1 = 0xBB67AE8584CAA73BULL;  // rng.py:21

__device__ __forceinline__ uint64_t philox4x64_word0(uint64_t seed, uint64_t stream,
                                                     uint64_t pos) {
    uint64_t c0 = pos, c1 = 0, c2 = stream, c3 = 0, k0 = seed, k1 = stream;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t lo0 = kPh64M0 * c0, hi0 = __umul64hi(kPh64M0, c0);
        const uint64_t lo1 = kPh64M1 * c2, hi1 = __umul64hi(kPh64M1, c2);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += kPh64W0;
        k1 += kPh64W1;
    }
    return c0;
}

// rng.py:64-67 / kernels.py:21-23: (w >> 11) * 2^-53, exact in FP64.
__device__ __forceinline__ double uniform53(uint64_t w) {
    return __dmul_rn((double)(w >> 11), 1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double stream_uniform(uint64_t seed, uint64_t stream,
                                                 uint64_t pos) {
    return uniform53(philox4x64_word0(seed, stream, pos));
}

// ---------------------------------------------------------- Philox4x32-10 --
constexpr uint32_t kPh32M0 = 0xD2511F53u;
constexpr uint32_t kPh32M1 = 0xCD9E8D57u;
constexpr uint32_t kPh32W0 = 0x9E3779B9u;
constexpr uint32_t kPh32W1 = 0xBB67AE85u;

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(kPh32M0, c.x), lo0 = kPh32M0 * c.x;
        const uint32_t hi1 = __umulhi(kPh32M1, c.z), lo1 = kPh32M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += kPh32W0;
        k1 += kPh32W1;
    }
    return c;
}

// Round keys of one Philox4x32-10 key, precomputed on the host and passed as a
// kernel parameter: the XORs then read them straight from the constant bank.
struct RoundKeys32 {
    uint32_t k0[10], k1[10];
};

inline RoundKeys32 make_round_keys32(uint64_t seed) {
    RoundKeys32 rk;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        rk.k0[r] = k0;
        rk.k1[r] = k1;
        k0 += kPh32W0;
        k1 += kPh32W1;
    }
    return rk;
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, const RoundKeys32& rk) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(kPh32M0, c.x), lo0 = kPh32M0 * c.x;
        const uint32_t hi1 = __umulhi(kPh32M1, c.z), lo1 = kPh32M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ rk.k0[r], lo1, hi0 ^ c.w ^ rk.k1[r], lo0);
    }
    return c;
}

}  // namespace ptmh

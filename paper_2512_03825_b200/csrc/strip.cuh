// strip.cuh -- the ferro strip update (J > 0, B = 0), shared by the
// checkerboard sweep kernels (checkerboard.cu) and the resident kernel's
// warp-owned lattices (resident.cu).  Described in checkerboard.cu above
// cb_half_sweep_ferro and in DESIGN.md section 4.
#pragma once
#include <cstdint>

#include "philox.cuh"

namespace ptmh {
namespace strip {
constexpr unsigned kFull = 0xffffffffu;
}

// base + esz * idx as one wide multiply-add (IMAD.WIDE.U32, FMA pipe) instead
// of the LEA / LEA.HI.X pair on the ALU pipe.  esz (= 4) is a kernel
// parameter so ptxas cannot strength-reduce the multiply into a shift.
template <typename T>
__device__ __forceinline__ T* word_at(T* base, uint32_t idx, uint32_t esz) {
    uint64_t r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(idx), "r"(esz), "l"((uint64_t)base));
    return reinterpret_cast<T*>(r);
}

// other-colour loads: the read-only path inside one launch, L2 (.cg) where
// another CTA of the same launch may have written the word (persistent path)
template <bool kNC>
__device__ __forceinline__ uint32_t ld_other(const uint32_t* p) {
    return kNC ? __ldg(p) : __ldcg(p);
}
// kTB == 2 (the colour-1 half of a temporally blocked item): the colour-0
// words this CTA stored before its barrier, read with ordinary (L1-allocating)
// loads -- coherent within the CTA after bar.sync; no other SM writes them
// while the item runs, and the item's acquire invalidated L1 after their
// last readers elsewhere
__device__ __forceinline__ uint32_t ld_cta(const uint32_t* p) {
    return __ldca(p);  // (explicit: a const __restrict__ pointer would be turned into the .nc path)
}
template <bool kNC, int kTB>
__device__ __forceinline__ uint32_t ld_oth(const uint32_t* p) {
    return kTB == 2 ? ld_cta(p) : ld_other<kNC>(p);
}

// One thread's strip: word column k of lattice rows i0 .. i0+kRows-1 of
// colour kColor.  kStats: colour 0 resets the lattice's stats, colour 1
// recomputes them -- the thread's (S, Bond) contributions in sumS / sumB,
// which the caller reduces (flush_stats).
//
// kTB: 0 = in place (packed is read and updated).  The temporally blocked
// persistent path (checkerboard.cu) runs a whole sweep of a band per item,
// out of place (ping-pong state buffers: `packed` holds sweep t-1, `out`
// receives sweep t, every word is stored): 1 = its colour-0 half (colour 1
// read from packed), 2 = its colour-1 half (colour 0 read from out, already
// updated by this CTA -- at L2, so kNC must be false -- except the rows just
// outside the band [band_lo, band_hi), which come from hup / hdn: the
// neighbouring bands' colour-0 words, recomputed by this CTA because those
// bands may be updating them concurrently; no stats reset in either half).
template <int kRows, int kColor, bool kStats, bool kNC, int kTB = 0>
__device__ __forceinline__ void ferro_strip(uint32_t* __restrict__ packed, int L, int WR, int64_t W,
                                            const int32_t* __restrict__ row_to_slot,
                                            const uint32_t* __restrict__ thresh, const RoundKeys32& rk,
                                            uint32_t ctr1, int64_t* __restrict__ stats, uint32_t esz,
                                            bool active, int64_t lat, int rem,
                                            uint32_t (&tie_m)[kRows][32], uint32_t (&tie_k4)[kRows][32],
                                            uint32_t (&tie_sn)[kRows][32],
                                            int& sumS, int& sumB, int wr_shift = -1,
                                            const uint32_t* __restrict__ planes = nullptr,
                                            uint32_t* __restrict__ out = nullptr, const uint32_t* hup = nullptr,
                                            const uint32_t* hdn = nullptr, int band_lo = 0, int band_hi = 0) {
    static_assert(kTB == 0 || (kTB == 1 && kColor == 0) || (kTB == 2 && kColor == 1), "kTB");
    const int lane = threadIdx.x & 31;
    const int strip = wr_shift >= 0 ? rem >> wr_shift : rem / WR;
    const int k = rem - strip * WR;
    const int i0 = strip * kRows;
    const uint32_t own_base = (uint32_t)((lat * 2 + kColor) * W);
    // where the own colour is stored (in place, or the next sweep's buffer)
    uint32_t* const dst = kTB ? out : packed;
    int slot = 0;
    uint32_t t3 = 0, t4 = 0;
    uint32_t tie_rows = 0;  // bit rr: row rr has ties
    if (active) {
        if (kTB == 0 && kColor == 0 && kStats && rem == 0) {  // colour-0 pass: reset, colour-1 pass recomputes
            stats[2 * lat] = 0;
            stats[2 * lat + 1] = 0;
        }
        const uint32_t* __restrict__ other = (kTB == 2 ? out : packed) + (lat * 2 + (1 - kColor)) * W;
        // (in place, own is own_dst: one __restrict__ pointer)
        uint32_t* __restrict__ own_dst = dst + own_base;
        const uint32_t* own = kTB ? packed + own_base : own_dst;
        // Threshold plane p of a site is bit p of t4 where K4 is set, else of
        // t3: Tm = K4 ? TB : TA with TA, TB in {0, ~0}.  Written as the
        // integer K4 * (TB - TA) - TA (TM[p] in {-1, 0, 1}, TC[p] = -TA) so
        // the select is one IMAD on the FMA pipe; the ALU pipe, which bounds
        // this kernel, only does the compare itself.  The persistent kernel
        // hands them over precomputed for the item's lattice (planes: TM[8],
        // TC[8], t3, t4, slot in shared memory).
        uint32_t TM[8], TC[8];
        if (planes) {
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                TM[p] = planes[p];
                TC[p] = planes[8 + p];
            }
            t3 = planes[16];
            t4 = planes[17];
            slot = (int)planes[18];
        } else {
            slot = row_to_slot[lat];
            t3 = __ldg(thresh + slot * 10 + 8);
            t4 = __ldg(thresh + slot * 10 + 9);
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                const uint32_t ta = (t3 >> (31 - p)) & 1u, tb = (t4 >> (31 - p)) & 1u;
                TM[p] = tb - ta;
                TC[p] = 0u - ta;
            }
        }
        const int kl = (k == 0) ? WR - 1 : k - 1;
        const int kr = (k == WR - 1) ? 0 : k + 1;
        // horizontal neighbour word column: kl when (i + colour) is even, else
        // kr; i0 is even, so row rr of the strip uses kl iff (rr + kColor) is
        // even.  Offsets are 32-bit word indices into one colour plane; the
        // next rows' offsets roll forward with one wrap (unsigned min) per row,
        // and addresses are formed with one wide IMAD (FMA pipe) each.
        const int dEven = kl - k, dOdd = kr - k;  // adjacent column, relative
        const uint32_t uWR = (uint32_t)WR, LW = (uint32_t)L * uWR;
        const uint32_t o0 = (uint32_t)(i0 * WR + k);
        uint32_t oup = o0 + LW - uWR;
        oup = min(oup, oup - LW);
        uint32_t o1 = o0 + uWR;
        o1 = min(o1, o1 - LW);
        // kTB == 2: rows band_lo - 1 and band_hi of the other colour come from hup / hdn
        const bool htop = kTB == 2 && i0 == band_lo, hbot = kTB == 2 && i0 + kRows == band_hi;
        uint32_t up = htop ? hup[k] : ld_oth<kNC, kTB>(word_at(other, oup, esz));
        uint32_t mid = ld_oth<kNC, kTB>(word_at(other, o0, esz));
        uint32_t dn = (kRows == 1 && hbot) ? hdn[k] : ld_oth<kNC, kTB>(word_at(other, o1, esz));
        uint32_t S = __ldcg(word_at(own, o0, esz));
        uint32_t adj = ld_oth<kNC, kTB>(word_at(other, o0 + (uint32_t)((kColor & 1) ? dOdd : dEven), esz));
        uint32_t o = o0;
        // strips of <= 8 rows unroll whole (a rank's C3 shard at 8 GPUs,
        // 4-row strips: 2.52 -> 2.65e12; at 4 GPUs, 8-row strips: 2.93 ->
        // 3.03e12); longer ones by 2 (by 4: C3 even, C4 -0.6 %, spills)
        constexpr int kUnroll = kRows <= 8 ? kRows : 2;
#pragma unroll kUnroll
        for (int rr = 0; rr < kRows; ++rr) {
            const bool even = ((rr + kColor) & 1) == 0;
            // prefetch row i+1 (own, adjacent) and row i+2 (other colour, below)
            uint32_t o2 = o1 + uWR;
            o2 = min(o2, o2 - LW);
            const uint32_t dn_n = (hbot && rr == kRows - 2) ? hdn[k] : ld_oth<kNC, kTB>(word_at(other, o2, esz));
            const uint32_t S_n = __ldcg(word_at(own, o1, esz));
            const uint32_t adj_n = ld_oth<kNC, kTB>(word_at(other, o1 + (uint32_t)(even ? dOdd : dEven), esz));
            const uint32_t hz = even ? __funnelshift_l(adj, mid, 1)   // m sees m-1
                                     : __funnelshift_r(mid, adj, 1);  // m sees m+1
            const uint32_t a = ~(S ^ up), b = ~(S ^ dn), c = ~(S ^ mid), d = ~(S ^ hz);
            const uint32_t s1 = a ^ b, c1 = a & b, s2 = c ^ d, c2 = c & d;
            const uint32_t k0 = s1 ^ s2, c3 = s1 & s2;
            const uint32_t k1 = c1 ^ c2 ^ c3, K4 = c1 & c2;
            const uint32_t upm = (k1 & k0) | K4;   // k = 3, 4
            const uint32_t K2 = k1 & ~k0;          // k = 2: dE = 0
            uint32_t acc = ~(k1 | K4);             // k = 0, 1: dE < 0
            const uint32_t w32 = o;
            const uint4 r0 = philox4x32_10(make_uint4(2u * w32, ctr1, (uint32_t)slot, 0u), rk);
            const uint4 r1 = philox4x32_10(make_uint4(2u * w32 + 1u, ctr1, (uint32_t)slot, 0u), rk);
            const uint32_t U[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
            acc |= K2 & ~U[0];  // neutral: u < 2^31 <=> top bit clear
            // byte compare u < t as the borrow of u - t, LSB plane first
            // (borrow' = MAJ(~u, t, borrow): one LOP3), plus the equality
            // chain for the ties; the per-site threshold plane is one IMAD
            uint32_t bor = 0, eq = upm;
#pragma unroll
            for (int p = 7; p >= 0; --p) {
                const uint32_t Tm = K4 * TM[p] + TC[p];
                bor = (~U[p] & Tm) | (~U[p] & bor) | (Tm & bor);
                eq &= ~(U[p] ^ Tm);
            }
            acc |= bor & upm;
            // ties (top byte equal): bookkeeping only, resolved after the loop
            tie_m[rr][lane] = eq;
            tie_k4[rr][lane] = K4;  // read at tie bits only
            if (kRows <= 16) tie_sn[rr][lane] = S ^ acc;  // the row's word as stored: the tie walk starts from it
            if (eq) tie_rows |= 1u << rr;
            const uint32_t Sn = S ^ acc;
            if (kTB || acc) __stcg(word_at(own_dst, o, esz), Sn);
            if (kColor == 1 && kStats) {
                // new aligned masks: a flip toggles alignment with all four neighbours
                const int kk = __popc(a ^ acc) + __popc(b ^ acc) + __popc(c ^ acc) + __popc(d ^ acc);
                sumB += 2 * kk - 128;                         // sum of s*nb = 2k - 4 per site
                sumS += 2 * (__popc(Sn) + __popc(mid)) - 64;  // both colours' words
            }
            up = mid;
            mid = dn;
            dn = dn_n;
            S = S_n;
            adj = adj_n;
            o = o1;
            o1 = o2;
        }
    }
    // ---- tie resolution: every lane walks its own ties (top byte equal)
    // across all its rows; the warp iterates max-ties-per-lane times.  The
    // lane owns its words, so accepted ties flip them with a plain
    // read-modify-write, and it accounts their (S, Bond) deltas itself.
    {
        int rr = -1;
        uint32_t m = 0, mk4 = 0, Sw = 0, w32 = 0;
        // sec24 < t24  <=>  word 0 < t24 << 8 (t << 8 drops the top byte)
        const uint32_t T3s = t3 << 8, T4s = t4 << 8;
        bool dirty = false;
        while (__any_sync(strip::kFull, tie_rows != 0 || m != 0)) {
            if (m == 0 && tie_rows != 0) {
                rr = __ffs(tie_rows) - 1;
                tie_rows &= tie_rows - 1;
                m = tie_m[rr][lane];
                mk4 = tie_k4[rr][lane];
                w32 = (uint32_t)((i0 + rr) * WR + k);
                // (shared memory: no L2 round trip per tie row; 32-row strips
                // keep only two scratch arrays to fit three CTAs per SM)
                Sw = kRows <= 16 ? tie_sn[rr][lane] : __ldcg(dst + own_base + w32);
                dirty = false;
            }
            if (m != 0) {
                const int bit = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t k4 = (mk4 >> bit) & 1u;
                const uint4 r2 =
                    philox4x32_10(make_uint4(w32 * 32u + (uint32_t)bit, ctr1, (uint32_t)slot, 1u), rk);
                if (r2.x < (k4 ? T4s : T3s)) {
                    if (kColor == 1 && kStats) {
                        sumS += ((Sw >> bit) & 1u) ? -2 : 2;
                        sumB += k4 ? -8 : -4;
                    }
                    Sw ^= 1u << bit;
                    dirty = true;
                }
                if (m == 0 && dirty) __stcg(dst + own_base + w32, Sw);
            }
        }
    }
}



}  // namespace ptmh

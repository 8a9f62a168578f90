// checkerboard.cu -- Mode F: multispin-coded checkerboard Metropolis sweep.
//
// Storage (HBM): per lattice, per colour c, the L*L/2 sites of that colour
// packed one bit per spin, half-lattice index h = i*(L/2) + (j>>1), bit
// (h & 31) of word (h >> 5).  For L % 64 == 0 a word never straddles a
// lattice row: word k of row i holds the colour-c sites m = 32k..32k+31.
//
// Neighbours of colour-c site (i, m) are colour-(1-c) sites: (i-1, m),
// (i+1, m), (i, m) and (i, m-1) if (i+c) is even else (i, m+1); in packed
// form the first three are whole words and the fourth is a funnel shift of
// two adjacent words.  One thread updates 32 sites per word with bitwise
// logic: the four "aligned neighbour" masks are summed bit-sliced, the site
// classes (s, nb) fall out as one-hot masks, and the acceptance test is a
// bit-sliced compare of 8 random planes against the class threshold's top
// byte, refined per site with 24 more random bits only on a tie
// (probability 2^-8).  The exact per-site definition is in DESIGN.md
// section 3 and oracle/ptmh_oracle.c (or_cb_u32, or_cb_sweep).
//
// The per-lattice reduction (kernel 2 of the north star) is fused: every
// accepted flip changes S = sum(s) by -2s and Bond = sum(s*(down+right)) by
// -2*s*nb = 8 - 4k (k = aligned neighbours); the thread sums these from
// popcounts of its bit-sliced masks, the warp reduces with shuffles and one
// 64-bit atomic per warp lands in the lattice's stats.  Integer sums are
// order-free, so the stats are deterministic.
#include <cuda_runtime.h>

#include "common.cuh"
#include "launchers.cuh"
#include "philox.cuh"

namespace ptmh {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr uint32_t kSymmetricFlag = 1u << 16;

// Uphill classes of the current configuration (host-built from always_mask).
struct ClassPlan {
    int n_up;
    int k[10];    // aligned-neighbour count 0..4
    int sf[10];   // 0: both spins, 1: s=+1 only, 2: s=-1 only
    int cls[10];  // column in the (R, 10) threshold table
};

__device__ __forceinline__ void decide_word(uint32_t S, uint32_t n1, uint32_t n2, uint32_t n3,
                                            uint32_t n4, uint32_t valid, uint32_t w,
                                            uint32_t h_base, int slot, uint32_t ctr1,
                                            const RoundKeys32& rk, const ClassPlan& plan,
                                            const uint32_t* __restrict__ thr_slot,
                                            uint32_t& acc_out, int& dS, int& dB) {
    // aligned-neighbour indicators and their bit-sliced sum k = k0 + 2 k1 + 4 k2
    const uint32_t a = ~(S ^ n1), b = ~(S ^ n2), c = ~(S ^ n3), d = ~(S ^ n4);
    const uint32_t s1 = a ^ b, c1 = a & b, s2 = c ^ d, c2 = c & d;
    const uint32_t k0 = s1 ^ s2, c3 = s1 & s2;
    const uint32_t k1 = c1 ^ c2 ^ c3, k2 = c1 & c2;
    uint32_t K[5];
    K[4] = k2;
    K[3] = k1 & k0;
    K[2] = k1 & ~k0;
    K[1] = k0 & ~k1;
    K[0] = ~(k0 | k1 | k2);

    uint32_t M[10];
    uint32_t thr[10];
    uint32_t uphill = 0;
#pragma unroll
    for (int q = 0; q < 10; ++q) {
        if (q < plan.n_up) {
            const uint32_t kq = K[plan.k[q]];
            const uint32_t sfm = plan.sf[q] == 0 ? 0xffffffffu : (plan.sf[q] == 1 ? S : ~S);
            M[q] = kq & sfm & valid;
            thr[q] = thr_slot[plan.cls[q]];
            uphill |= M[q];
        } else {
            M[q] = 0;
            thr[q] = 0;
        }
    }
    uint32_t acc = valid & ~uphill;  // dE <= 0: always accepted
    if (uphill) {
        const uint4 r0 = philox4x32_10(make_uint4(2u * w, ctr1, (uint32_t)slot, 0u), rk);
        const uint4 r1 = philox4x32_10(make_uint4(2u * w + 1u, ctr1, (uint32_t)slot, 0u), rk);
        const uint32_t U[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
        uint32_t lt = 0, eq = uphill;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            uint32_t Tm = 0;
#pragma unroll
            for (int q = 0; q < 10; ++q)
                if (q < plan.n_up) Tm |= M[q] & (0u - ((thr[q] >> (31 - p)) & 1u));
            lt |= eq & ~U[p] & Tm;
            eq &= ~(U[p] ^ Tm);
        }
        acc |= lt;
        // ties on the top byte: compare the low 24 bits with a per-site draw
        while (eq) {
            const int bit = __ffs(eq) - 1;
            eq &= eq - 1;
            uint32_t t24 = 0;
#pragma unroll
            for (int q = 0; q < 10; ++q)
                if (q < plan.n_up && ((M[q] >> bit) & 1u)) t24 = thr[q] & 0x00ffffffu;
            const uint4 r2 = philox4x32_10(make_uint4(h_base + (uint32_t)bit, ctr1, (uint32_t)slot, 1u), rk);
            if ((r2.x >> 8) < t24) acc |= 1u << bit;
        }
    }
    acc_out = acc;
    // fused reduction: dS = sum(-2 s), dBond = sum(8 - 4 k) over flips
    dS += 2 * (__popc(acc & ~S) - __popc(acc & S));
    dB += 8 * __popc(acc) - 4 * (__popc(acc & k0) + 2 * __popc(acc & k1) + 4 * __popc(acc & k2));
}

__device__ __forceinline__ void flush_stats(int64_t* stats, int64_t lat, bool active, int dS, int dB) {
    const int64_t lat0 = __shfl_sync(kFullMask, lat, 0);
    const bool uniform = __all_sync(kFullMask, (lat == lat0) || !active);
    if (uniform) {
        for (int o = 16; o > 0; o >>= 1) {
            dS += __shfl_down_sync(kFullMask, dS, o);
            dB += __shfl_down_sync(kFullMask, dB, o);
        }
        if ((threadIdx.x & 31) == 0) {
            if (dS) atomicAdd((unsigned long long*)&stats[2 * lat0], (unsigned long long)(long long)dS);
            if (dB) atomicAdd((unsigned long long*)&stats[2 * lat0 + 1], (unsigned long long)(long long)dB);
        }
    } else if (active) {
        if (dS) atomicAdd((unsigned long long*)&stats[2 * lat], (unsigned long long)(long long)dS);
        if (dB) atomicAdd((unsigned long long*)&stats[2 * lat + 1], (unsigned long long)(long long)dB);
    }
}

// --------------------------------------------------- fast path, L % 64 == 0 --
// One thread: word column k of a strip of kRows lattice rows.  The colour-(1-c)
// column k for rows i0-1 .. i0+kRows is held in registers (vertical reuse).
template <int kRows>
__global__ void __launch_bounds__(256) cb_half_sweep_fast(
    uint32_t* __restrict__ packed, int64_t rows, int L, int WR, int64_t W,
    const int32_t* __restrict__ row_to_slot, const uint32_t* __restrict__ thresh, ClassPlan plan,
    const RoundKeys32 rk, uint32_t ctr1, int color, int64_t* __restrict__ stats) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int strips = L / kRows;
    const int64_t per_lat = (int64_t)strips * WR;
    const bool active = tid < rows * per_lat;
    const int64_t lat = active ? tid / per_lat : 0;
    const int rem = (int)(tid - lat * per_lat);
    const int strip = rem / WR;
    const int k = rem - strip * WR;
    int dS = 0, dB = 0;
    if (active) {
        const uint32_t* __restrict__ other = packed + (lat * 2 + (1 - color)) * W;
        uint32_t* __restrict__ own = packed + (lat * 2 + color) * W;
        const int slot = row_to_slot[lat];
        const uint32_t* thr_slot = thresh + (int64_t)slot * 10;
        const int i0 = strip * kRows;
        const int kl = (k == 0) ? WR - 1 : k - 1;
        const int kr = (k == WR - 1) ? 0 : k + 1;
        uint32_t O[kRows + 2];
#pragma unroll
        for (int r = 0; r < kRows + 2; ++r) {
            int i = i0 - 1 + r;
            i = (i < 0) ? i + L : (i >= L ? i - L : i);
            O[r] = __ldg(other + (int64_t)i * WR + k);
        }
#pragma unroll
        for (int rr = 0; rr < kRows; ++rr) {
            const int i = i0 + rr;
            const int64_t wi = (int64_t)i * WR + k;
            const uint32_t S = own[wi];
            const uint32_t mid = O[rr + 1];
            uint32_t hz;
            if (((i + color) & 1) == 0) {
                const uint32_t adj = __ldg(other + (int64_t)i * WR + kl);
                hz = __funnelshift_l(adj, mid, 1);  // site m sees m-1
            } else {
                const uint32_t adj = __ldg(other + (int64_t)i * WR + kr);
                hz = __funnelshift_r(mid, adj, 1);  // site m sees m+1
            }
            uint32_t acc;
            decide_word(S, O[rr], O[rr + 2], mid, hz, 0xffffffffu, (uint32_t)wi, (uint32_t)(wi * 32),
                        slot, ctr1, rk, plan, thr_slot, acc, dS, dB);
            if (acc) own[wi] = S ^ acc;
        }
    }
    flush_stats(stats, lat, active, dS, dB);
}

// ------------------------------------ fast path, J > 0 and B = 0 (ferro) --
// The benchmark and paper setting.  k = 0, 1 aligned neighbours (dE < 0) are
// always accepted, k = 2 (dE = 0) with probability 1/2 (u < 2^31: random
// plane 0 clear), k = 3 (dE = 4J) and k = 4 (dE = 8J) against thresholds
// t3 = thr[slot][8], t4 = thr[slot][9] for both spin signs, so the per-site
// threshold plane is a select on K4.
//
// Rows are walked with a rolling window of the other colour's words (one new
// load per row).  Ties on the top random byte are queued per warp in shared
// memory and resolved 32 per secondary-Philox pass after the row loop; an
// accepted tie flips its spin with atomicXor (the owner already stored the
// word).  Statistics: the colour-0 pass zeroes the lattice's (S, Bond); the
// colour-1 pass recomputes them from the new configuration -- S from both
// colours' words, Bond = sum over colour-1 sites of s*nb (every bond has
// exactly one colour-1 end) -- plus the deltas of its own tie flips.
#ifndef PTMH_FERRO_MINB
#define PTMH_FERRO_MINB 1
#endif

template <int kRows, bool kStats>
__global__ void __launch_bounds__(256, PTMH_FERRO_MINB) cb_half_sweep_ferro(
    uint32_t* __restrict__ packed, int64_t rows, int L, int WR, int64_t W,
    const int32_t* __restrict__ row_to_slot, const uint32_t* __restrict__ thresh, const RoundKeys32 rk,
    uint32_t ctr1, int color, int64_t* __restrict__ stats) {
    constexpr int kWarps = 8;
    __shared__ uint32_t tie_m[kWarps][kRows][32], tie_k4[kWarps][kRows][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int strips = L / kRows;
    const int64_t per_lat = (int64_t)strips * WR;
    const bool active = tid < rows * per_lat;
    const int64_t lat = active ? tid / per_lat : 0;
    const int rem = (int)(tid - lat * per_lat);
    const int strip = rem / WR;
    const int k = rem - strip * WR;
    const int i0 = strip * kRows;
    const uint32_t own_base = (uint32_t)((lat * 2 + color) * W);
    int slot = 0;
    uint32_t t3 = 0, t4 = 0;
    int sumS = 0, sumB = 0;
    uint32_t tie_rows = 0;  // bit rr: row rr has ties
    if (active) {
        if (!kStats && rem == 0) {  // colour-0 pass: reset, colour-1 pass recomputes
            stats[2 * lat] = 0;
            stats[2 * lat + 1] = 0;
        }
        const uint32_t* __restrict__ other = packed + (lat * 2 + (1 - color)) * W;
        uint32_t* __restrict__ own = packed + own_base;
        slot = row_to_slot[lat];
        t3 = __ldg(thresh + slot * 10 + 8);
        t4 = __ldg(thresh + slot * 10 + 9);
        uint32_t TA[8], TB[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            TA[p] = 0u - ((t3 >> (31 - p)) & 1u);
            TB[p] = 0u - ((t4 >> (31 - p)) & 1u);
        }
        const int kl = (k == 0) ? WR - 1 : k - 1;
        const int kr = (k == WR - 1) ? 0 : k + 1;
        // horizontal neighbour word column: kl when (i + colour) is even, else kr
        const int kadj0 = ((i0 + color) & 1) == 0 ? kl : kr;
        const int kadj1 = ((i0 + color) & 1) == 0 ? kr : kl;
        uint32_t up = __ldg(other + (i0 == 0 ? L - 1 : i0 - 1) * WR + k);
        uint32_t mid = __ldg(other + i0 * WR + k);
        uint32_t dn = __ldg(other + (i0 + 1 == L ? 0 : i0 + 1) * WR + k);
        uint32_t S = own[i0 * WR + k];
        uint32_t adj = __ldg(other + i0 * WR + kadj0);
#pragma unroll 2
        for (int rr = 0; rr < kRows; ++rr) {
            const int i = i0 + rr;
            const int row = i * WR;
            // prefetch row i+1 (own, adjacent) and row i+2 (other colour, below)
            const int i1 = (i + 1 == L) ? 0 : i + 1;
            const int i2 = (i1 + 1 == L) ? 0 : i1 + 1;
            const uint32_t dn_n = __ldg(other + i2 * WR + k);
            const uint32_t S_n = own[i1 * WR + k];
            const uint32_t adj_n = __ldg(other + i1 * WR + ((rr & 1) ? kadj0 : kadj1));
            const uint32_t hz = (((i + color) & 1) == 0) ? __funnelshift_l(adj, mid, 1)   // m sees m-1
                                                         : __funnelshift_r(mid, adj, 1);  // m sees m+1
            const uint32_t a = ~(S ^ up), b = ~(S ^ dn), c = ~(S ^ mid), d = ~(S ^ hz);
            const uint32_t s1 = a ^ b, c1 = a & b, s2 = c ^ d, c2 = c & d;
            const uint32_t k0 = s1 ^ s2, c3 = s1 & s2;
            const uint32_t k1 = c1 ^ c2 ^ c3, K4 = c1 & c2;
            const uint32_t upm = (k1 & k0) | K4;   // k = 3, 4
            const uint32_t K2 = k1 & ~k0;          // k = 2: dE = 0
            uint32_t acc = ~(k1 | K4);             // k = 0, 1: dE < 0
            const uint32_t w32 = (uint32_t)(row + k);
            const uint4 r0 = philox4x32_10(make_uint4(2u * w32, ctr1, (uint32_t)slot, 0u), rk);
            const uint4 r1 = philox4x32_10(make_uint4(2u * w32 + 1u, ctr1, (uint32_t)slot, 0u), rk);
            const uint32_t U[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
            acc |= K2 & ~U[0];  // neutral: u < 2^31 <=> top bit clear
            // byte compare u < t as the borrow of u - t, LSB plane first
            // (borrow' = MAJ(~u, t, borrow): one LOP3), plus the equality
            // chain for the ties; K4 pinned in a register so the per-site
            // threshold plane is a single select
            uint32_t K4r = K4;
            asm volatile("" : "+r"(K4r));
            uint32_t bor = 0, eq = upm;
#pragma unroll
            for (int p = 7; p >= 0; --p) {
                const uint32_t Tm = (K4r & TB[p]) | (~K4r & TA[p]);
                bor = (~U[p] & Tm) | (~U[p] & bor) | (Tm & bor);
                eq &= ~(U[p] ^ Tm);
            }
            acc |= bor & upm;
            // ties (top byte equal): bookkeeping only, resolved after the loop
            tie_m[warp][rr][lane] = eq;
            tie_k4[warp][rr][lane] = eq & K4;
            tie_rows |= (eq != 0u ? 1u : 0u) << rr;
            const uint32_t Sn = S ^ acc;
            if (acc) own[row + k] = Sn;
            if (kStats) {
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
        }
    }
    // ---- tie resolution: every lane walks its own ties (top byte equal)
    // across all its rows; the warp iterates max-ties-per-lane times.  The
    // lane owns its words, so accepted ties flip them with a plain
    // read-modify-write, and it accounts their (S, Bond) deltas itself.
    {
        int rr = -1;
        uint32_t m = 0, mk4 = 0, Sw = 0, w32 = 0;
        bool dirty = false;
        while (__any_sync(kFullMask, tie_rows != 0 || m != 0)) {
            if (m == 0 && tie_rows != 0) {
                rr = __ffs(tie_rows) - 1;
                tie_rows &= tie_rows - 1;
                m = tie_m[warp][rr][lane];
                mk4 = tie_k4[warp][rr][lane];
                w32 = (uint32_t)((i0 + rr) * WR + k);
                Sw = packed[own_base + w32];
                dirty = false;
            }
            if (m != 0) {
                const int bit = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t k4 = (mk4 >> bit) & 1u;
                const uint32_t t24 = (k4 ? t4 : t3) & 0x00ffffffu;
                const uint4 r2 =
                    philox4x32_10(make_uint4(w32 * 32u + (uint32_t)bit, ctr1, (uint32_t)slot, 1u), rk);
                if ((r2.x >> 8) < t24) {
                    if (kStats) {
                        sumS += ((Sw >> bit) & 1u) ? -2 : 2;
                        sumB += k4 ? -8 : -4;
                    }
                    Sw ^= 1u << bit;
                    dirty = true;
                }
                if (m == 0 && dirty) packed[own_base + w32] = Sw;
            }
        }
    }
    if (kStats) flush_stats(stats, lat, active, sumS, sumB);
}

// ------------------------------------------------------- generic even L --
__device__ __forceinline__ uint32_t get_bit(const uint32_t* p, int64_t h) {
    return (__ldg(p + (h >> 5)) >> (h & 31)) & 1u;
}

__global__ void __launch_bounds__(256) cb_half_sweep_generic(
    uint32_t* __restrict__ packed, int64_t rows, int L, int64_t W,
    const int32_t* __restrict__ row_to_slot, const uint32_t* __restrict__ thresh, ClassPlan plan,
    const RoundKeys32 rk, uint32_t ctr1, int color, int64_t* __restrict__ stats) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = tid < rows * W;
    const int64_t lat = active ? tid / W : 0;
    const int64_t w = tid - lat * W;
    int dS = 0, dB = 0;
    if (active) {
        const int Lh = L / 2;
        const int64_t H = (int64_t)L * Lh;
        const uint32_t* other = packed + (lat * 2 + (1 - color)) * W;
        uint32_t* own = packed + (lat * 2 + color) * W;
        const int slot = row_to_slot[lat];
        uint32_t n1 = 0, n2 = 0, n3 = 0, n4 = 0, valid = 0;
        for (int b = 0; b < 32; ++b) {
            const int64_t h = w * 32 + b;
            if (h >= H) break;
            valid |= 1u << b;
            const int i = (int)(h / Lh);
            const int m = (int)(h - (int64_t)i * Lh);
            const int j = 2 * m + ((i + color) & 1);
            const int iu = (i == 0) ? L - 1 : i - 1;
            const int id = (i == L - 1) ? 0 : i + 1;
            const int jl = (j == 0) ? L - 1 : j - 1;
            const int jr = (j == L - 1) ? 0 : j + 1;
            n1 |= get_bit(other, (int64_t)iu * Lh + (j >> 1)) << b;
            n2 |= get_bit(other, (int64_t)id * Lh + (j >> 1)) << b;
            n3 |= get_bit(other, (int64_t)i * Lh + (jl >> 1)) << b;
            n4 |= get_bit(other, (int64_t)i * Lh + (jr >> 1)) << b;
        }
        const uint32_t S = own[w];
        uint32_t acc;
        decide_word(S, n1, n2, n3, n4, valid, (uint32_t)w, (uint32_t)(w * 32), slot, ctr1, rk,
                    plan, thresh + (int64_t)slot * 10, acc, dS, dB);
        if (acc) own[w] = S ^ acc;
    }
    flush_stats(stats, lat, active, dS, dB);
}

// --------------------------------------------------------- pack / unpack --
__global__ void cb_pack_kernel(const int8_t* __restrict__ spins, int64_t rows, int L, int64_t W,
                               uint32_t* __restrict__ packed) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= rows * 2 * W) return;
    const int64_t lat = tid / (2 * W);
    const int64_t rem = tid - lat * 2 * W;
    const int color = (int)(rem / W);
    const int64_t w = rem - (int64_t)color * W;
    const int Lh = L / 2;
    const int64_t H = (int64_t)L * Lh;
    const int8_t* s = spins + lat * (int64_t)L * L;
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b) {
        const int64_t h = w * 32 + b;
        if (h >= H) break;
        const int i = (int)(h / Lh);
        const int m = (int)(h - (int64_t)i * Lh);
        const int j = 2 * m + ((i + color) & 1);
        word |= (uint32_t)(s[(int64_t)i * L + j] > 0) << b;
    }
    packed[tid] = word;
}

__global__ void cb_unpack_kernel(const uint32_t* __restrict__ packed, int64_t rows, int L, int64_t W,
                                 int8_t* __restrict__ spins) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = (int64_t)L * L;
    if (tid >= rows * n) return;
    const int64_t lat = tid / n;
    const int64_t site = tid - lat * n;
    const int i = (int)(site / L), j = (int)(site - (int64_t)i * L);
    const int color = (i + j) & 1;
    const int64_t h = (int64_t)i * (L / 2) + (j >> 1);
    const uint32_t bit = (packed[(lat * 2 + color) * W + (h >> 5)] >> (h & 31)) & 1u;
    spins[tid] = bit ? 1 : -1;
}

// lattices in slot order: out[k] = lattice slot_to_row[k] (full_states recording)
__global__ void cb_unpack_slots_kernel(const uint32_t* __restrict__ packed, const int64_t* __restrict__ s2r,
                                       int64_t R, int L, int64_t W, int8_t* __restrict__ out) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = (int64_t)L * L;
    if (tid >= R * n) return;
    const int64_t k = tid / n, site = tid - k * n;
    const int64_t lat = s2r[k];
    const int i = (int)(site / L), j = (int)(site - (int64_t)i * L);
    const int color = (i + j) & 1;
    const int64_t h = (int64_t)i * (L / 2) + (j >> 1);
    out[tid] = ((packed[(lat * 2 + color) * W + (h >> 5)] >> (h & 31)) & 1u) ? 1 : -1;
}

// Audit reduction from the packed state: S over both colours, Bond as the sum
// over colour-0 sites of s*nb = 2k - 4 (every bond has one colour-0 end).
__global__ void cb_row_stats_kernel(const uint32_t* __restrict__ packed, int64_t rows, int L, int64_t W,
                                    int64_t* __restrict__ stats) {
    const int64_t lat = blockIdx.x;
    const int Lh = L / 2;
    const int64_t H = (int64_t)L * Lh;
    const uint32_t* c0 = packed + lat * 2 * W;
    const uint32_t* c1 = c0 + W;
    long long S = 0, Bd = 0;
    for (int64_t w = threadIdx.x; w < W; w += blockDim.x) {
        uint32_t n1 = 0, n2 = 0, n3 = 0, n4 = 0, valid = 0;
        for (int b = 0; b < 32; ++b) {
            const int64_t h = w * 32 + b;
            if (h >= H) break;
            valid |= 1u << b;
            const int i = (int)(h / Lh);
            const int m = (int)(h - (int64_t)i * Lh);
            const int j = 2 * m + (i & 1);
            const int iu = (i == 0) ? L - 1 : i - 1;
            const int id = (i == L - 1) ? 0 : i + 1;
            const int jl = (j == 0) ? L - 1 : j - 1;
            const int jr = (j == L - 1) ? 0 : j + 1;
            n1 |= get_bit(c1, (int64_t)iu * Lh + (j >> 1)) << b;
            n2 |= get_bit(c1, (int64_t)id * Lh + (j >> 1)) << b;
            n3 |= get_bit(c1, (int64_t)i * Lh + (jl >> 1)) << b;
            n4 |= get_bit(c1, (int64_t)i * Lh + (jr >> 1)) << b;
        }
        const uint32_t s = c0[w];
        const uint32_t a = ~(s ^ n1), b2 = ~(s ^ n2), c = ~(s ^ n3), d = ~(s ^ n4);
        const int nv = __popc(valid);
        const int ksum = __popc(a & valid) + __popc(b2 & valid) + __popc(c & valid) + __popc(d & valid);
        Bd += 2 * ksum - 4 * nv;
        S += 2 * __popc(s & valid) - nv + 2 * __popc(c1[w] & valid) - nv;
    }
    for (int o = 16; o > 0; o >>= 1) {
        S += __shfl_down_sync(kFullMask, S, o);
        Bd += __shfl_down_sync(kFullMask, Bd, o);
    }
    __shared__ long long sS[32], sB[32];
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { sS[wid] = S; sB[wid] = Bd; }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long a = 0, b = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { a += sS[k]; b += sB[k]; }
        stats[2 * lat] = a;
        stats[2 * lat + 1] = b;
    }
}

// energies / observables by slot from per-lattice stats (lattice.py:61-65)
__global__ void cb_slot_energy_kernel(const int64_t* __restrict__ stats, const int64_t* __restrict__ s2r,
                                      int64_t R, double J, double B, double* __restrict__ energies,
                                      int64_t* __restrict__ sums) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= R) return;
    const int64_t row = s2r[k];
    const int64_t S = stats[2 * row], Bd = stats[2 * row + 1];
    energies[k] = __dsub_rn(__dmul_rn(B, (double)S), __dmul_rn(J, (double)Bd));
    sums[k] = S;
}

__global__ void cb_observe_kernel(const int64_t* __restrict__ stats, const int64_t* __restrict__ s2r,
                                  int64_t R, double nsites, double J, double B, double* __restrict__ obs_e,
                                  double* __restrict__ obs_m, int64_t ncols, int64_t col) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= R) return;
    const int64_t row = s2r[k];
    const int64_t S = stats[2 * row], Bd = stats[2 * row + 1];
    obs_e[k * ncols + col] = __dsub_rn(__dmul_rn(B, (double)S), __dmul_rn(J, (double)Bd));
    obs_m[k * ncols + col] = __ddiv_rn((double)S, nsites);
}

// ------------------------------------------------------------ launchers --
int64_t cb_words(int64_t L) { return (L * L / 2 + 31) / 32; }

static ClassPlan make_plan(uint32_t always_mask) {
    ClassPlan p{};
    const bool sym = (always_mask & kSymmetricFlag) != 0;
    for (int k = 0; k <= 4; ++k) {
        const int cp = 5 + k, cm = 4 - k;
        const bool ap = (always_mask >> cp) & 1u, am = (always_mask >> cm) & 1u;
        if (sym && !ap && !am) {
            p.k[p.n_up] = k; p.sf[p.n_up] = 0; p.cls[p.n_up] = cp; ++p.n_up;
            continue;
        }
        if (!ap) { p.k[p.n_up] = k; p.sf[p.n_up] = 1; p.cls[p.n_up] = cp; ++p.n_up; }
        if (!am) { p.k[p.n_up] = k; p.sf[p.n_up] = 2; p.cls[p.n_up] = cm; ++p.n_up; }
    }
    return p;
}

void fill_class_plan(uint32_t always_mask, int* n_up, int* k, int* sf, int* cls, int* ferro) {
    const ClassPlan p = make_plan(always_mask);
    *n_up = p.n_up;
    for (int q = 0; q < 10; ++q) {
        k[q] = p.k[q];
        sf[q] = p.sf[q];
        cls[q] = p.cls[q];
    }
    *ferro = (always_mask & kSymmetricFlag) && (always_mask & 0x3ffu) == 0x078u;
}

#ifndef PTMH_FERRO_ROWS
#define PTMH_FERRO_ROWS 8
#endif
constexpr int kFastRows = PTMH_FERRO_ROWS;

int launch_cb_sweeps(uint32_t* packed, int64_t rows, int64_t L, const int32_t* row_to_slot,
                     const uint32_t* thresh, uint32_t always_mask, uint64_t seed, int64_t first_sweep,
                     int64_t n_sweeps, int64_t* stats, cudaStream_t s) {
    if (rows == 0 || n_sweeps == 0) return PTMH_OK;
    const ClassPlan plan = make_plan(always_mask);
    const RoundKeys32 rk = make_round_keys32(seed);
    const int64_t W = cb_words(L);
    const bool fast = (L % 64) == 0 && (L % kFastRows) == 0;
    // symmetric thresholds, k <= 1 always, k = 2 neutral (1/2), k = 3, 4 uphill
    const bool ferro = (always_mask & kSymmetricFlag) && (always_mask & 0x3ffu) == 0x078u &&
                       rows * 2 * W < (1LL << 32);  // 32-bit word offsets in the tie queue
    for (int64_t t = first_sweep; t < first_sweep + n_sweeps; ++t) {
        for (int color = 0; color < 2; ++color) {
            const uint32_t ctr1 = (uint32_t)(2 * t + color);
            if (fast && ferro && L >= 1024) {  // long rows: amortise the per-thread setup over 16
                const int WR = (int)(L / 64);
                const int64_t threads = rows * (L / 16) * WR;
                if (color == 0)
                    cb_half_sweep_ferro<16, false><<<ceil_div(threads, 256), 256, 0, s>>>(
                        packed, rows, (int)L, WR, W, row_to_slot, thresh, rk, ctr1, color, stats);
                else
                    cb_half_sweep_ferro<16, true><<<ceil_div(threads, 256), 256, 0, s>>>(
                        packed, rows, (int)L, WR, W, row_to_slot, thresh, rk, ctr1, color, stats);
            } else if (fast && ferro) {
                const int WR = (int)(L / 64);
                const int64_t threads = rows * (L / kFastRows) * WR;
                if (color == 0)
                    cb_half_sweep_ferro<kFastRows, false><<<ceil_div(threads, 256), 256, 0, s>>>(
                        packed, rows, (int)L, WR, W, row_to_slot, thresh, rk, ctr1, color, stats);
                else
                    cb_half_sweep_ferro<kFastRows, true><<<ceil_div(threads, 256), 256, 0, s>>>(
                        packed, rows, (int)L, WR, W, row_to_slot, thresh, rk, ctr1, color, stats);
            } else if (fast) {
                const int WR = (int)(L / 64);
                const int64_t threads = rows * (L / kFastRows) * WR;
                cb_half_sweep_fast<kFastRows><<<ceil_div(threads, 256), 256, 0, s>>>(
                    packed, rows, (int)L, WR, W, row_to_slot, thresh, plan, rk, ctr1, color,
                    stats);
            } else {
                const int64_t threads = rows * W;
                cb_half_sweep_generic<<<ceil_div(threads, 256), 256, 0, s>>>(
                    packed, rows, (int)L, W, row_to_slot, thresh, plan, rk, ctr1, color, stats);
            }
            PTMH_LAUNCH_CHECK();
        }
    }
    return PTMH_OK;
}

int launch_cb_pack(const int8_t* spins, int64_t rows, int64_t L, uint32_t* packed, cudaStream_t s) {
    const int64_t W = cb_words(L), n = rows * 2 * W;
    if (n == 0) return PTMH_OK;
    cb_pack_kernel<<<ceil_div(n, 256), 256, 0, s>>>(spins, rows, (int)L, W, packed);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_cb_unpack(const uint32_t* packed, int64_t rows, int64_t L, int8_t* spins, cudaStream_t s) {
    const int64_t W = cb_words(L), n = rows * L * L;
    if (n == 0) return PTMH_OK;
    cb_unpack_kernel<<<ceil_div(n, 256), 256, 0, s>>>(packed, rows, (int)L, W, spins);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_cb_unpack_slots(const uint32_t* packed, const int64_t* s2r, int64_t R, int64_t L, int8_t* out,
                           cudaStream_t s) {
    const int64_t n = R * L * L;
    if (n == 0) return PTMH_OK;
    cb_unpack_slots_kernel<<<ceil_div(n, 256), 256, 0, s>>>(packed, s2r, R, (int)L, cb_words(L), out);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_cb_row_stats(const uint32_t* packed, int64_t rows, int64_t L, int64_t* stats, cudaStream_t s) {
    if (rows == 0) return PTMH_OK;
    cb_row_stats_kernel<<<(unsigned)rows, 256, 0, s>>>(packed, rows, (int)L, cb_words(L), stats);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_cb_slot_energies(const int64_t* stats, const int64_t* s2r, int64_t R, double J, double B,
                            double* energies, int64_t* sums, cudaStream_t s) {
    if (R == 0) return PTMH_OK;
    cb_slot_energy_kernel<<<ceil_div(R, 256), 256, 0, s>>>(stats, s2r, R, J, B, energies, sums);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_cb_observe(const int64_t* stats, const int64_t* s2r, int64_t R, int64_t L, double J, double B,
                      double* obs_e, double* obs_m, int64_t ncols, int64_t col, cudaStream_t s) {
    if (R == 0) return PTMH_OK;
    cb_observe_kernel<<<ceil_div(R, 256), 256, 0, s>>>(stats, s2r, R, (double)(L * L), J, B, obs_e, obs_m,
                                                      ncols, col);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

}  // namespace ptmh

// resident_reg.cu -- the resident run (sweeps + exchange rounds in one
// cooperative launch, as resident.cu) for 64^2 and 32^2 ferro lattices held
// in REGISTERS: one warp owns one lattice for the whole launch (C5: 4096
// lattices of 64^2, C1: 8 of 32^2, a round every sweep).
//
// A 64^2 lattice is 64 rows x 2 colours x one 32-site word (L % 64 == 0, WR =
// 1).  Lane l keeps rows 2l and 2l+1 of both colours in four registers.  A
// half-sweep of colour c needs the other colour's rows 2l-1 .. 2l+2: two of
// them are the lane's own, the other two come from lanes l-1 and l+1 by one
// shuffle each; the horizontal neighbour is the same row's word rotated by one
// site (a row is one word, periodic).  So a sweep touches no memory at all:
// the strip code of resident.cu (cb_resident_p2p_kernel, 2-row strips read
// from L1/L2) spent ~40 % of its instructions on the loads, stores, address
// arithmetic and the tie bookkeeping in shared memory.  The update itself --
// bit-sliced classes, two Philox4x32-10 blocks per word, the byte compare
// against the threshold planes, one tie walk per lane and half-sweep -- is
// strip.cuh's, with the same counters: bit-exact with oracle/ptmh_oracle.c.
// Exchange rounds are resident.cu's point-to-point rounds (rounds.cuh).
#include <cooperative_groups.h>
#include <cstdlib>
#include <cuda_runtime.h>

#include "common.cuh"
#include "launchers.cuh"
#include "philox.cuh"
#include "rounds.cuh"

namespace ptmh {

namespace {
constexpr unsigned kAll = 0xffffffffu;
}

// the threshold-plane select coefficients of thresholds t3, t4 (strip.cuh:
// Tm = K4 * TM + TC)
__device__ __forceinline__ void reg64_planes(uint32_t t3, uint32_t t4, uint32_t (&TM)[8], uint32_t (&TC)[8]) {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        const uint32_t ta = (t3 >> (31 - p)) & 1u, tb = (t4 >> (31 - p)) & 1u;
        TM[p] = tb - ta;
        TC[p] = 0u - ta;
    }
}

// One half-sweep of colour kColor of the warp's lattice.  C[c][rr]: colour c,
// row 2*lane + rr.  kStats: the colour-1 pass also returns the lane's (S, Bond)
// contributions of the new configuration (strip.cuh's formulas).
template <int kColor, bool kStats>
__device__ __forceinline__ void reg64_pass(uint32_t (&C)[2][2], const uint32_t (&TM)[8], const uint32_t (&TC)[8],
                                           uint32_t t3, uint32_t t4, uint32_t slot, const RoundKeys32& rk,
                                           uint32_t ctr1, int lane, int& sumS, int& sumB) {
    const uint32_t o0 = C[1 - kColor][0], o1 = C[1 - kColor][1];
    const uint32_t above = __shfl_sync(kAll, o1, (lane + 31) & 31);  // other colour, row 2l - 1
    const uint32_t below = __shfl_sync(kAll, o0, (lane + 1) & 31);   // other colour, row 2l + 2
    uint32_t eqm[2], k4m[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const uint32_t w32 = (uint32_t)(2 * lane + rr);  // the row = the word's index in its colour plane
        const bool even = ((rr + kColor) & 1) == 0;      // (row + colour) even: site m sees m - 1
        const uint32_t S = C[kColor][rr];
        const uint32_t mid = rr == 0 ? o0 : o1;
        const uint32_t up = rr == 0 ? above : o0;
        const uint32_t dn = rr == 0 ? o1 : below;
        const uint32_t hz = even ? __funnelshift_l(mid, mid, 1) : __funnelshift_r(mid, mid, 1);
        const uint32_t a = ~(S ^ up), b = ~(S ^ dn), c = ~(S ^ mid), d = ~(S ^ hz);
        const uint32_t s1 = a ^ b, c1 = a & b, s2 = c ^ d, c2 = c & d;
        const uint32_t k0 = s1 ^ s2, c3 = s1 & s2;
        const uint32_t k1 = c1 ^ c2 ^ c3, K4 = c1 & c2;
        const uint32_t upm = (k1 & k0) | K4;  // k = 3, 4
        const uint32_t K2 = k1 & ~k0;         // k = 2: dE = 0
        uint32_t acc = ~(k1 | K4);            // k = 0, 1: dE < 0
        const uint4 r0 = philox4x32_10(make_uint4(2u * w32, ctr1, slot, 0u), rk);
        const uint4 r1 = philox4x32_10(make_uint4(2u * w32 + 1u, ctr1, slot, 0u), rk);
        const uint32_t U[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
        acc |= K2 & ~U[0];
        uint32_t bor = 0, eq = upm;
#pragma unroll
        for (int p = 7; p >= 0; --p) {
            const uint32_t Tm = K4 * TM[p] + TC[p];
            bor = (~U[p] & Tm) | (~U[p] & bor) | (Tm & bor);
            eq &= ~(U[p] ^ Tm);
        }
        acc |= bor & upm;
        const uint32_t Sn = S ^ acc;
        C[kColor][rr] = Sn;
        eqm[rr] = eq;
        k4m[rr] = K4;
        if (kStats) {
            const int kk = __popc(a ^ acc) + __popc(b ^ acc) + __popc(c ^ acc) + __popc(d ^ acc);
            sumB += 2 * kk - 128;
            sumS += 2 * (__popc(Sn) + __popc(mid)) - 64;
        }
    }
    // ties (top byte equal): each lane walks its own; the warp iterates
    // max-ties-per-lane times.  sec24 < t24 <=> word 0 < t24 << 8
    const uint32_t T3s = t3 << 8, T4s = t4 << 8;
    while (__any_sync(kAll, (eqm[0] | eqm[1]) != 0)) {
        const int rr = eqm[0] ? 0 : 1;
        const uint32_t m = rr ? eqm[1] : eqm[0];
        if (m != 0) {
            const int bit = __ffs(m) - 1;
            if (rr) eqm[1] &= eqm[1] - 1; else eqm[0] &= eqm[0] - 1;
            const uint32_t k4 = ((rr ? k4m[1] : k4m[0]) >> bit) & 1u;
            const uint32_t w32 = (uint32_t)(2 * lane + rr);
            const uint4 r2 = philox4x32_10(make_uint4(w32 * 32u + (uint32_t)bit, ctr1, slot, 1u), rk);
            if (r2.x < (k4 ? T4s : T3s)) {
                const uint32_t Sw = rr ? C[kColor][1] : C[kColor][0];
                if (kStats) {
                    sumS += ((Sw >> bit) & 1u) ? -2 : 2;
                    sumB += k4 ? -8 : -4;
                }
                if (rr) C[kColor][1] = Sw ^ (1u << bit); else C[kColor][0] = Sw ^ (1u << bit);
            }
        }
    }
}

// The round's partner-independent inputs, loaded after the publish so that
// their latency overlaps the partner's word in flight (loading them before
// the sweep, held in registers across it, measured slower at C5: 6.55 ->
// 6.80 us).
struct RoundIn {
    double u, bi, bj;
    uint32_t ot3, ot4;
    __device__ void load(const ResidentArgs& A, int R, int64_t round, int k) {
        const int first = (int)(round & 1), n_pairs = (R - first) / 2;
        if (k < first || (k - first) / 2 >= n_pairs) return;
        const int p = (k - first) / 2, i = first + 2 * p, other = k == i ? i + 1 : i;
        u = A.u_table[(round - A.u_round0) * A.u_stride + p];
        bi = A.betas[i];
        bj = A.betas[i + 1];
        ot3 = __ldg(A.thresh + other * 10 + 8);
        ot4 = __ldg(A.thresh + other * 10 + 9);
    }
};

// Lane 0 of a warp that owns a lattice, after a sweep whose (S, Bond) it
// holds: the final stats, the observables by slot and the point-to-point
// round (resident.cu, rounds.cuh); nk / n3 / n4 receive the lattice's slot
// and thresholds for the next sweep.
// local: the ring is in the CTA's shared memory (every lattice of the run in
// one CTA), so the round word is a volatile shared store / poll.
__device__ __forceinline__ void reg_round(const ResidentArgs& A, uint64_t* ring, int R, bool multi, bool local,
                                          int row, int64_t round, int64_t col, bool rec, bool exch, bool last, int k,
                                          int64_t S, int64_t Bd, int& nk, uint32_t& n3, uint32_t& n4) {
    static_assert((kRing & (kRing - 1)) == 0, "ring depth: a power of two");
    uint64_t* const slot_word = ring + (round & (kRing - 1)) * (int64_t)R;
    if (exch) {  // first: the partner is waiting for it
        const uint64_t mine = p2p_pack(S, Bd, round);
        if (local) {
            *reinterpret_cast<volatile uint64_t*>(slot_word + k) = mine;
        } else if (multi) {
            for (int g = 0; g < A.world; ++g)
                st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(A.pub_peer[g]) + (slot_word - ring) + k,
                                   mine);
        } else {
            st_relaxed_u64(slot_word + k, mine);
        }
    }
    if (last) {
        A.stats[2 * row] = S;
        A.stats[2 * row + 1] = Bd;
    }
    if (rec) {  // by slot, before the round (executor.py order)
        A.obs_e[(int64_t)k * A.ncols + col] = __dsub_rn(__dmul_rn(A.B, (double)S), __dmul_rn(A.J, (double)Bd));
        A.obs_m[(int64_t)k * A.ncols + col] = __ddiv_rn((double)S, (double)A.L * A.L);
    }
    const int first = (int)(round & 1), n_pairs = (R - first) / 2;
    if (exch && k >= first && (k - first) / 2 < n_pairs) {
        // everything that does not need the partner's energy, while its word travels
        const int p = (k - first) / 2, i = first + 2 * p, other = k == i ? i + 1 : i;
        RoundIn in;
        in.load(A, R, round, k);
        const double u = in.u, bi = in.bi, bj = in.bj;
        const uint32_t ot3 = in.ot3, ot4 = in.ot4;
        const uint64_t want = (uint64_t)((round & 0x7fff) | 0x8000);
        auto poll = [&]() -> uint64_t {
            if (local) return *reinterpret_cast<volatile const uint64_t*>(slot_word + other);
            return multi ? ld_relaxed_sys_u64(slot_word + other) : ld_relaxed_u64(slot_word + other);
        };
        uint64_t v = poll();
        while ((v & 0xffffull) != want) {
            if (!local) __nanosleep(64);
            v = poll();
        }
        const int64_t So = p2p_field(v, 16), Bo = p2p_field(v, 40);
        const int64_t Si = k == i ? S : So, Bi = k == i ? Bd : Bo;
        const int64_t Sj = k == i ? So : S, Bj = k == i ? Bo : Bd;
        const double Ei = __dsub_rn(__dmul_rn(A.B, (double)Si), __dmul_rn(A.J, (double)Bi));
        const double Ej = __dsub_rn(__dmul_rn(A.B, (double)Sj), __dmul_rn(A.J, (double)Bj));
        bool near = false;
        const bool acc = swap_decide(__dsub_rn(bi, bj), Ei, Ej, u, near);
        if (k == i) {
            if (acc) atomicAdd((unsigned long long*)&A.counters[0], 1ull);
            if (near) atomicAdd((unsigned long long*)&A.counters[1], 1ull);
        }
        if (acc) {
            nk = other;
            n3 = ot3;
            n4 = ot4;
        }
    }
}

template <int kThreads>
__global__ void __launch_bounds__(kThreads) cb_resident_reg64_kernel(ResidentArgs A) {
    const int lane = threadIdx.x & 31, wq = (int)threadIdx.x >> 5;
    const bool multi = A.world > 1;
    const int R = multi ? A.R_total : A.R;  // slots (pairs, swap streams, ring entries)
    __shared__ unsigned long long s_ring[kRing * 32];  // local: the round words of <= 32 lattices
    const bool local = A.local_ring != 0;
    if (local) {
        for (int i = threadIdx.x; i < kRing * 32; i += blockDim.x) s_ring[i] = 0ull;
        __syncthreads();
    }
    const int lo = (int)((int64_t)A.R * blockIdx.x / gridDim.x);
    const int hi = (int)((int64_t)A.R * (blockIdx.x + 1) / gridDim.x);
    if (wq >= hi - lo) return;  // no block-wide barrier below: spare warps leave
    const int row = lo + wq;
    uint32_t* const gl = A.packed + (int64_t)row * 2 * 64;
    uint32_t C[2][2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const uint2 v = *reinterpret_cast<const uint2*>(gl + c * 64 + 2 * lane);
        C[c][0] = v.x;
        C[c][1] = v.y;
    }
    uint64_t* const ring = local ? reinterpret_cast<uint64_t*>(s_ring)
                                 : reinterpret_cast<uint64_t*>(A.slot_stats);  // kRing x R words
    int k = A.r2s[A.buf][row];
    uint32_t t3 = __ldg(A.thresh + k * 10 + 8), t4 = __ldg(A.thresh + k * 10 + 9);
    uint32_t TM[8], TC[8];
    reg64_planes(t3, t4, TM, TC);
    int rounds = 0;
    RunSchedule sx, sr;
    sx.init(A.swap_every, A.first_sweep + 1);
    sr.init(A.record_every, A.first_sweep + 1);
    for (int64_t t = A.first_sweep; t < A.first_sweep + A.n_sweeps; ++t, sx.step(), sr.step()) {
        const int64_t done = t + 1;
        const bool rec = sr.hit();
        const bool exch = sx.hit() && done < A.total_sweeps;
        const bool last = t + 1 == A.first_sweep + A.n_sweeps;
        const bool need_stats = rec || exch || last;
        int sS = 0, sB = 0;
        reg64_pass<0, false>(C, TM, TC, t3, t4, (uint32_t)k, A.rk, (uint32_t)(2 * t), lane, sS, sB);
        if (need_stats)
            reg64_pass<1, true>(C, TM, TC, t3, t4, (uint32_t)k, A.rk, (uint32_t)(2 * t + 1), lane, sS, sB);
        else
            reg64_pass<1, false>(C, TM, TC, t3, t4, (uint32_t)k, A.rk, (uint32_t)(2 * t + 1), lane, sS, sB);
        if (!need_stats) continue;
        sS = __reduce_add_sync(kAll, sS);
        sB = __reduce_add_sync(kAll, sB);
        int nk = k;
        uint32_t n3 = t3, n4 = t4;
        if (lane == 0)
            reg_round(A, ring, R, multi, local, row, exch ? sx.index() : 0, sr.index(), rec, exch, last, k,
                      (int64_t)sS, (int64_t)sB, nk, n3, n4);
        if (exch) ++rounds;
        const int k_new = __shfl_sync(kAll, nk, 0);
        if (k_new != k) {  // (warp-uniform) the new slot's thresholds
            k = k_new;
            t3 = __shfl_sync(kAll, n3, 0);
            t4 = __shfl_sync(kAll, n4, 0);
            reg64_planes(t3, t4, TM, TC);
        }
    }
#pragma unroll
    for (int c = 0; c < 2; ++c)
        *reinterpret_cast<uint2*>(gl + c * 64 + 2 * lane) = make_uint2(C[c][0], C[c][1]);
    // the permutation is an output only: the final mapping, in the buffer the
    // grid-barrier kernel would leave it in (buf flips once per round)
    if (lane == 0) {
        const int fb = A.buf ^ (rounds & 1);
        A.r2s[fb][row] = k;
        A.s2r[fb][k] = A.row_lo + row;
    }
}

// 64^2 ferro lattices (W = 64 words per colour, one per row), one warp each,
// every lattice's warp resident at once.  Returns 1 when it does not apply.
int launch_cb_resident_reg64(const ResidentArgs& a, int grid, int threads, cudaStream_t s) {
    const char* e = getenv("PTMH_RESIDENT_REG");  // "0": resident.cu's strip kernel (A/B)
    if (e && e[0] == '0') return 1;
    if (!a.ferro || a.L != 64 || a.WR != 1 || a.W != 64 || (a.swap_every > 0 && !a.u_table)) return 1;
    const char* ep = getenv("PTMH_RESIDENT_P2P");  // "0": grid-barrier rounds (resident.cu)
    if (ep && ep[0] == '0' && a.swap_every > 0) return 1;
    if (threads > 1024 || (int64_t)(a.R + grid - 1) / grid > threads / 32) return 1;
    if (a.swap_every > 0 && a.world == 1) PTMH_CUDA(cudaMemsetAsync(a.slot_stats, 0, (size_t)kRing * a.R * 8, s));
    void* kargs[] = {const_cast<ResidentArgs*>(&a)};
    // C5's CTAs hold 28 lattices (896 threads): the 896-thread build may use
    // 72 registers instead of 64 (PTMH_RESIDENT_REG896=0: the 1024 build, A/B)
    const char* e9 = getenv("PTMH_RESIDENT_REG896");
    const void* fn = threads <= 896 && !(e9 && e9[0] == '0') ? (const void*)cb_resident_reg64_kernel<896>
                                                              : (const void*)cb_resident_reg64_kernel<1024>;
    PTMH_CUDA(cudaLaunchCooperativeKernel(fn, grid, threads, kargs, 0, s));
    cb_set_last_launch(CbLaunchInfo{9, 2, threads, 1, 0, grid});
    return PTMH_OK;
}

// ---------------------------------------------------------------- 32^2 --
// C1 (8 lattices of 32^2): a colour plane is 16 words, word w holding rows 2w
// (bits 0-15) and 2w+1 (bits 16-31) as two 16-site segments.  Lane l < 16 of
// the owning warp keeps word l of both colours; the rows above and below a
// segment come from the neighbouring segment of the same word or of words
// l -+ 1 (one shuffle each), the horizontal neighbour is a rotation within the
// segment (resident.cu's kGatherSegments gather, on registers).  Without the
// loads, a half-sweep no longer waits for the other colour's words just
// stored by the other lanes to come back from L2.
// Both colours' random planes of a sweep in one go: lanes 0-15 draw colour
// 0's (counter 2t), lanes 16-31, which hold no words, colour 1's (2t + 1) for
// the same word; the colour-1 pass takes them with a shuffle (the planes do
// not depend on the spins, and the slot only changes at the round after the
// sweep).  C1: 1.20 -> 1.00 us per sweep without rounds.
__device__ __forceinline__ void reg32_planes(uint32_t slot, const RoundKeys32& rk, uint32_t ctr0, int lane,
                                             uint32_t (&U)[8]) {
    const uint32_t w32 = (uint32_t)(lane & 15), c = ctr0 + (uint32_t)(lane >> 4);
    const uint4 r0 = philox4x32_10(make_uint4(2u * w32, c, slot, 0u), rk);
    const uint4 r1 = philox4x32_10(make_uint4(2u * w32 + 1u, c, slot, 0u), rk);
    U[0] = r0.x; U[1] = r0.y; U[2] = r0.z; U[3] = r0.w;
    U[4] = r1.x; U[5] = r1.y; U[6] = r1.z; U[7] = r1.w;
}

template <int kColor, bool kStats>
__device__ __forceinline__ void reg32_pass(uint32_t (&C)[2], const uint32_t (&TM)[8], const uint32_t (&TC)[8],
                                           uint32_t t3, uint32_t t4, uint32_t slot, const RoundKeys32& rk,
                                           uint32_t ctr1, int lane, int& sumS, int& sumB, const uint32_t (&U)[8]) {
    constexpr uint32_t kLo = 0x00010001u, kHi = 0x80008000u;  // bit 0 / bit 15 of each segment
    // segments with (row + colour) even: the row-2w segment for colour 0
    constexpr uint32_t kEven = kColor ? 0xffff0000u : 0x0000ffffu;
    const int w = lane & 15;
    const uint32_t mid = C[1 - kColor];
    const uint32_t prev = __shfl_sync(kAll, mid, (w + 15) & 15);
    const uint32_t next = __shfl_sync(kAll, mid, (w + 1) & 15);
    const uint32_t S = C[kColor];
    const uint32_t up = __funnelshift_l(prev, mid, 16);  // row above each segment
    const uint32_t dn = __funnelshift_r(mid, next, 16);  // row below
    const uint32_t rot_l = ((mid << 1) & ~kLo) | ((mid >> 15) & kLo);  // site m - 1
    const uint32_t rot_r = ((mid >> 1) & ~kHi) | ((mid << 15) & kHi);  // site m + 1
    const uint32_t hz = (rot_l & kEven) | (rot_r & ~kEven);
    const uint32_t a = ~(S ^ up), b = ~(S ^ dn), c = ~(S ^ mid), d = ~(S ^ hz);
    const uint32_t s1 = a ^ b, c1 = a & b, s2 = c ^ d, c2 = c & d;
    const uint32_t k0 = s1 ^ s2, c3 = s1 & s2;
    const uint32_t k1 = c1 ^ c2 ^ c3, K4 = c1 & c2;
    const uint32_t upm = (k1 & k0) | K4, K2 = k1 & ~k0;
    uint32_t acc = ~(k1 | K4);
    const uint32_t w32 = (uint32_t)w;
    acc |= K2 & ~U[0];
    uint32_t bor = 0, eq = upm;
#pragma unroll
    for (int p = 7; p >= 0; --p) {
        const uint32_t Tm = K4 * TM[p] + TC[p];
        bor = (~U[p] & Tm) | (~U[p] & bor) | (Tm & bor);
        eq &= ~(U[p] ^ Tm);
    }
    acc |= bor & upm;
    uint32_t Sn = S ^ acc;
    if (kStats) {
        const int kk = __popc(a ^ acc) + __popc(b ^ acc) + __popc(c ^ acc) + __popc(d ^ acc);
        sumB += 2 * kk - 128;
        sumS += 2 * (__popc(Sn) + __popc(mid)) - 64;
    }
    if (lane >= 16) eq = 0;  // (lanes 16-31 hold no words: no ties to walk)
    while (__any_sync(kAll, eq != 0)) {
        if (eq != 0) {
            const int bit = __ffs(eq) - 1;
            eq &= eq - 1;
            const uint32_t k4 = (K4 >> bit) & 1u;
            const uint4 r2 = philox4x32_10(make_uint4(w32 * 32u + (uint32_t)bit, ctr1, slot, 1u), rk);
            if (r2.x < ((k4 ? t4 : t3) << 8)) {  // sec24 < t24 <=> word 0 < t24 << 8
                if (kStats) {
                    sumS += ((Sn >> bit) & 1u) ? -2 : 2;
                    sumB += k4 ? -8 : -4;
                }
                Sn ^= 1u << bit;
            }
        }
    }
    if (lane < 16) C[kColor] = Sn;
}

template <int kThreads>
__global__ void __launch_bounds__(kThreads) cb_resident_reg32_kernel(ResidentArgs A) {
    const int lane = threadIdx.x & 31, wq = (int)threadIdx.x >> 5;
    const bool multi = A.world > 1;
    const int R = multi ? A.R_total : A.R;
    __shared__ unsigned long long s_ring[kRing * 32];  // local: the round words of <= 32 lattices
    const bool local = A.local_ring != 0;
    if (local) {
        for (int i = threadIdx.x; i < kRing * 32; i += blockDim.x) s_ring[i] = 0ull;
        __syncthreads();
    }
    const int lo = (int)((int64_t)A.R * blockIdx.x / gridDim.x);
    const int hi = (int)((int64_t)A.R * (blockIdx.x + 1) / gridDim.x);
    if (wq >= hi - lo) return;  // no block-wide barrier below: spare warps leave
    const int row = lo + wq;
    uint32_t* const gl = A.packed + (int64_t)row * 2 * 16;
    uint32_t C[2];
    C[0] = lane < 16 ? gl[lane] : 0u;
    C[1] = lane < 16 ? gl[16 + lane] : 0u;
    uint64_t* const ring = local ? reinterpret_cast<uint64_t*>(s_ring)
                                 : reinterpret_cast<uint64_t*>(A.slot_stats);  // kRing x R words
    int k = A.r2s[A.buf][row];
    uint32_t t3 = __ldg(A.thresh + k * 10 + 8), t4 = __ldg(A.thresh + k * 10 + 9);
    uint32_t TM[8], TC[8];
    reg64_planes(t3, t4, TM, TC);
    int rounds = 0;
    RunSchedule sx, sr;
    sx.init(A.swap_every, A.first_sweep + 1);
    sr.init(A.record_every, A.first_sweep + 1);
    for (int64_t t = A.first_sweep; t < A.first_sweep + A.n_sweeps; ++t, sx.step(), sr.step()) {
        const int64_t done = t + 1;
        const bool rec = sr.hit();
        const bool exch = sx.hit() && done < A.total_sweeps;
        const bool last = t + 1 == A.first_sweep + A.n_sweeps;
        const bool need_stats = rec || exch || last;
        int sS = 0, sB = 0;
        uint32_t U[8], U1[8];
        reg32_planes((uint32_t)k, A.rk, (uint32_t)(2 * t), lane, U);
#pragma unroll
        for (int p = 0; p < 8; ++p) U1[p] = __shfl_down_sync(kAll, U[p], 16);
        reg32_pass<0, false>(C, TM, TC, t3, t4, (uint32_t)k, A.rk, (uint32_t)(2 * t), lane, sS, sB, U);
        if (need_stats)
            reg32_pass<1, true>(C, TM, TC, t3, t4, (uint32_t)k, A.rk, (uint32_t)(2 * t + 1), lane, sS, sB, U1);
        else
            reg32_pass<1, false>(C, TM, TC, t3, t4, (uint32_t)k, A.rk, (uint32_t)(2 * t + 1), lane, sS, sB, U1);
        if (!need_stats) continue;
        if (lane >= 16) sS = sB = 0;  // (idle lanes computed on zero words)
        sS = __reduce_add_sync(kAll, sS);
        sB = __reduce_add_sync(kAll, sB);
        int nk = k;
        uint32_t n3 = t3, n4 = t4;
        if (lane == 0)
            reg_round(A, ring, R, multi, local, row, exch ? sx.index() : 0, sr.index(), rec, exch, last, k,
                      (int64_t)sS, (int64_t)sB, nk, n3, n4);
        if (exch) ++rounds;
        const int k_new = __shfl_sync(kAll, nk, 0);
        if (k_new != k) {
            k = k_new;
            t3 = __shfl_sync(kAll, n3, 0);
            t4 = __shfl_sync(kAll, n4, 0);
            reg64_planes(t3, t4, TM, TC);
        }
    }
    if (lane < 16) {
        gl[lane] = C[0];
        gl[16 + lane] = C[1];
    }
    if (lane == 0) {
        const int fb = A.buf ^ (rounds & 1);
        A.r2s[fb][row] = k;
        A.s2r[fb][k] = A.row_lo + row;
    }
}

// 32^2 ferro lattices (16 words per colour), one warp each; returns 1 when
// it does not apply
int launch_cb_resident_reg32(const ResidentArgs& a, int grid, int threads, cudaStream_t s) {
    const char* e = getenv("PTMH_RESIDENT_REG");  // "0": resident.cu's kernels (A/B)
    if (e && e[0] == '0') return 1;
    if (!a.ferro || a.L != 32 || a.W != 16 || (a.swap_every > 0 && !a.u_table)) return 1;
    const char* ep = getenv("PTMH_RESIDENT_P2P");
    if (ep && ep[0] == '0' && a.swap_every > 0) return 1;
    if (threads > 1024 || (int64_t)(a.R + grid - 1) / grid > threads / 32) return 1;
    // up to 32 lattices on one GPU (C1: 8): ONE CTA with the round words in
    // its shared memory -- a round is then a shared store and poll, where
    // the L2 ring took ~1 us of the 2.4 us sweep + round (PTMH_RESIDENT_LOCALRING=0: off)
    const char* el = getenv("PTMH_RESIDENT_LOCALRING");
    ResidentArgs args = a;
    args.local_ring = a.world == 1 && a.R <= 32 && !(el && el[0] == '0');
    const int g = args.local_ring ? 1 : grid, th = args.local_ring ? 32 * a.R : threads;
    if (a.swap_every > 0 && a.world == 1 && !args.local_ring)
        PTMH_CUDA(cudaMemsetAsync(a.slot_stats, 0, (size_t)kRing * a.R * 8, s));
    void* kargs[] = {&args};
    // (up to 8 lattices in one CTA: a 256-thread build without the 64-register cap)
    const void* fn = th <= 256 ? (const void*)cb_resident_reg32_kernel<256> : (const void*)cb_resident_reg32_kernel<1024>;
    PTMH_CUDA(cudaLaunchCooperativeKernel(fn, g, th, kargs, 0, s));
    cb_set_last_launch(CbLaunchInfo{10, args.local_ring ? 0 : 1, th, 1, 0, g});
    return PTMH_OK;
}

}  // namespace ptmh

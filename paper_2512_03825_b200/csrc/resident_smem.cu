// resident_smem.cu -- the resident run (sweeps + exchange rounds in one
// cooperative launch, as resident.cu) for lattices owned by thread-block
// CLUSTERS that hold the lattice in SHARED MEMORY for the whole launch.
//
// C2 (64 lattices of 256^2, a round every sweep) has fewer lattices than SMs
// and too few words per lattice for the sweep kernels; resident.cu's cluster
// kernel read its words from L2 after every cluster barrier (each barrier's
// acquire invalidates L1) and updated one word per thread, so a tie anywhere
// in a warp cost the whole warp a secondary Philox block per word
// (ncu: ~345 thread-instructions per word, 14 % warps active, IPC 1.4).
//
// Here a cluster of cs CTAs owns one lattice; CTA rank q keeps rows
// [q*band, (q+1)*band) of both colours (band = L/cs) in its shared memory,
// and reads the two halo rows straight from its neighbours' shared memory
// (DSMEM).  A thread runs the sweep kernels' strip update (strip.cuh's
// arithmetic: rolling window, bit-sliced classes, byte compare, one tie walk
// per strip) on kRows-row strips.  The cluster barrier separates the
// colours; the colour-1 pass recomputes (S, Bond), reduced per warp into the
// CTA's partial, which every CTA of the cluster sums over DSMEM.  Rounds are
// point to point (resident.cu, cb_resident_p2p_kernel): rank 0 publishes the
// lattice's round word, every CTA polls the partner slot's word and decides
// the pair redundantly (same inputs, same rule), so no grid barrier runs.
//
// Same chain and random numbers as checkerboard.cu / resident.cu (bit-exact
// with oracle/ptmh_oracle.c): the Philox counters use the global word index
// i*WR + k of the colour plane.
#include <cooperative_groups.h>
#include <cstdlib>
#include <cuda_runtime.h>

#include "common.cuh"
#include "launchers.cuh"
#include "philox.cuh"
#include "rounds.cuh"

namespace cg = cooperative_groups;

namespace ptmh {

namespace {
constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kNotApplicable = 1;
}  // namespace

// Shared-memory layout of a band: plane c at c * BW (BW = band * WR words);
// row rl = sr * kRows + rr, word column k at  rr * NS + sr * WR + k  where
// NS = band / kRows * WR is the number of strips.  Strip s = sr * WR + k is
// thread s's, so for a fixed rr the lanes of a warp touch consecutive words
// (no bank conflicts), and the strip's rows are NS words apart.
template <int kRows>
__device__ __forceinline__ int band_word(int rl, int k, int WR, int NS) {
    return (rl % kRows) * NS + (rl / kRows) * WR + k;
}

// One thread's strip s of colour kColor: rows band_lo + sr*kRows .. +kRows-1,
// word column k.  own / oth: this CTA's planes; up_row / dn_row: the other
// colour's row above / below the band (a neighbour CTA's shared memory, or
// this CTA's own when the cluster is one CTA), as word-column arrays.
// The strip's random planes (two Philox4x32-10 blocks per row word).  They
// do not depend on the spins, so the kernel draws them ahead of the pass
// where a thread owns one strip (smem_draws below): between the arrive and
// the wait of the cluster barrier before the pass, and during the round for
// the next sweep's colour 0.
template <int kRows>
__device__ __forceinline__ void smem_draws(int s, int WR, int wr_shift, int band_lo, uint32_t slot,
                                           const RoundKeys32& rk, uint32_t ctr1, uint32_t (&U)[kRows][8]) {
    const int sr = wr_shift >= 0 ? s >> wr_shift : s / WR;
    const int k = s - sr * WR;
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) {
        const uint32_t w32 = (uint32_t)((band_lo + sr * kRows + rr) * WR + k);
        const uint4 r0 = philox4x32_10(make_uint4(2u * w32, ctr1, slot, 0u), rk);
        const uint4 r1 = philox4x32_10(make_uint4(2u * w32 + 1u, ctr1, slot, 0u), rk);
        U[rr][0] = r0.x;
        U[rr][1] = r0.y;
        U[rr][2] = r0.z;
        U[rr][3] = r0.w;
        U[rr][4] = r1.x;
        U[rr][5] = r1.y;
        U[rr][6] = r1.z;
        U[rr][7] = r1.w;
    }
}

// ties (top byte equal): the lane walks its own, the warp iterates
// max-ties-per-lane times (strip.cuh)
template <int kRows, bool kStats>
__device__ __forceinline__ void smem_ties(uint32_t* __restrict__ own, int s, int WR, int NS, int i0, int k,
                                          uint32_t tie_rows, uint32_t t3, uint32_t t4, uint32_t slot,
                                          const RoundKeys32& rk, uint32_t ctr1, uint32_t (&tie_m)[kRows][32],
                                          uint32_t (&tie_k4)[kRows][32], uint32_t (&tie_sn)[kRows][32],
                                          int& sumS, int& sumB) {
    const int lane = threadIdx.x & 31;
    int rr = -1;
    uint32_t m = 0, mk4 = 0, Sw = 0, w32 = 0;
    bool dirty = false;
    while (__any_sync(kFullMask, tie_rows != 0 || m != 0)) {
        if (m == 0 && tie_rows != 0) {
            rr = __ffs(tie_rows) - 1;
            tie_rows &= tie_rows - 1;
            m = tie_m[rr][lane];
            mk4 = tie_k4[rr][lane];
            Sw = tie_sn[rr][lane];
            w32 = (uint32_t)((i0 + rr) * WR + k);
            dirty = false;
        }
        if (m != 0) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t k4 = (mk4 >> bit) & 1u;
            const uint4 r2 = philox4x32_10(make_uint4(w32 * 32u + (uint32_t)bit, ctr1, slot, 1u), rk);
            if (r2.x < ((k4 ? t4 : t3) << 8)) {  // sec24 < t24 <=> word 0 < t24 << 8
                if (kStats) {
                    sumS += ((Sw >> bit) & 1u) ? -2 : 2;
                    sumB += k4 ? -8 : -4;
                }
                Sw ^= 1u << bit;
                dirty = true;
            }
            if (m == 0 && dirty) own[rr * NS + s] = Sw;
        }
    }
}

template <int kRows, int kColor, bool kStats, bool kPre = false>
__device__ __forceinline__ void smem_strip(uint32_t* __restrict__ own, const uint32_t* __restrict__ oth,
                                           const uint32_t* up_row, const uint32_t* dn_row, int s, int WR,
                                           int wr_shift, int NS, int band_lo, const uint32_t (&TM)[8],
                                           const uint32_t (&TC)[8], uint32_t t3, uint32_t t4, uint32_t slot,
                                           const RoundKeys32& rk, uint32_t ctr1, uint32_t (&tie_m)[kRows][32],
                                           uint32_t (&tie_k4)[kRows][32], uint32_t (&tie_sn)[kRows][32],
                                           int& sumS, int& sumB, const uint32_t (*Upre)[8] = nullptr) {
    const int lane = threadIdx.x & 31;
    const int sr = wr_shift >= 0 ? s >> wr_shift : s / WR;
    const int k = s - sr * WR;
    const bool top = sr == 0, bottom = s >= NS - WR;
    const int kl = (k == 0) ? WR - 1 : k - 1;
    const int kr = (k == WR - 1) ? 0 : k + 1;
    const int i0 = band_lo + sr * kRows;
    uint32_t up = top ? up_row[k] : oth[(kRows - 1) * NS + s - WR];
    uint32_t mid = oth[s];
    uint32_t tie_rows = 0;
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) {
        const int i = i0 + rr;
        const bool even = ((i + kColor) & 1) == 0;
        const uint32_t dn = rr + 1 < kRows ? oth[(rr + 1) * NS + s] : (bottom ? dn_row[k] : oth[s + WR]);
        const uint32_t adj = oth[rr * NS + s - k + (even ? kl : kr)];
        const uint32_t S = own[rr * NS + s];
        const uint32_t hz = even ? __funnelshift_l(adj, mid, 1)   // m sees m-1
                                 : __funnelshift_r(mid, adj, 1);  // m sees m+1
        const uint32_t a = ~(S ^ up), b = ~(S ^ dn), c = ~(S ^ mid), d = ~(S ^ hz);
        const uint32_t s1 = a ^ b, c1 = a & b, s2 = c ^ d, c2 = c & d;
        const uint32_t k0 = s1 ^ s2, c3 = s1 & s2;
        const uint32_t k1 = c1 ^ c2 ^ c3, K4 = c1 & c2;
        const uint32_t upm = (k1 & k0) | K4;  // k = 3, 4
        const uint32_t K2 = k1 & ~k0;         // k = 2: dE = 0
        uint32_t acc = ~(k1 | K4);            // k = 0, 1: dE < 0
        uint32_t U[8];
        if constexpr (kPre) {
#pragma unroll
            for (int p = 0; p < 8; ++p) U[p] = Upre[rr][p];
        } else {
            const uint32_t w32 = (uint32_t)(i * WR + k);
            const uint4 r0 = philox4x32_10(make_uint4(2u * w32, ctr1, slot, 0u), rk);
            const uint4 r1 = philox4x32_10(make_uint4(2u * w32 + 1u, ctr1, slot, 0u), rk);
            U[0] = r0.x; U[1] = r0.y; U[2] = r0.z; U[3] = r0.w;
            U[4] = r1.x; U[5] = r1.y; U[6] = r1.z; U[7] = r1.w;
        }
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
        tie_m[rr][lane] = eq;
        tie_k4[rr][lane] = K4;
        tie_sn[rr][lane] = Sn;
        if (eq) tie_rows |= 1u << rr;
        if (acc) own[rr * NS + s] = Sn;
        if (kStats) {
            const int kk = __popc(a ^ acc) + __popc(b ^ acc) + __popc(c ^ acc) + __popc(d ^ acc);
            sumB += 2 * kk - 128;
            sumS += 2 * (__popc(Sn) + __popc(mid)) - 64;
        }
        up = mid;
        mid = dn;
    }
    smem_ties<kRows, kStats>(own, s, WR, NS, i0, k, tie_rows, t3, t4, slot, rk, ctr1, tie_m, tie_k4, tie_sn, sumS,
                             sumB);
}

// the threshold-plane select coefficients of slot k (strip.cuh: Tm = K4 * TM + TC)
__device__ __forceinline__ void smem_set_slot(int k, uint32_t t3, uint32_t t4,
                                              uint32_t* s_mask) {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        const uint32_t ta = (t3 >> (31 - p)) & 1u, tb = (t4 >> (31 - p)) & 1u;
        s_mask[p] = tb - ta;
        s_mask[8 + p] = 0u - ta;
    }
    s_mask[16] = t3;
    s_mask[17] = t4;
    s_mask[18] = (uint32_t)k;
}

template <int kRows, int kThreads, int kColor, bool kStats, bool kPre = false>
__device__ __forceinline__ void smem_pass(const ResidentArgs& A, uint32_t* s_lat, const uint32_t* up_pl,
                                          const uint32_t* dn_pl, int BW, int NS, int band_lo, int wr_shift,
                                          const uint32_t* s_mask, uint32_t ctr1,
                                          uint32_t (&s_tie)[kThreads / 32][3][kRows][32], int& sS, int& sB,
                                          const uint32_t (*Upre)[8] = nullptr) {
    uint32_t TM[8], TC[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        TM[p] = s_mask[p];
        TC[p] = s_mask[8 + p];
    }
    const uint32_t t3 = s_mask[16], t4 = s_mask[17], slot = s_mask[18];
    const int WR = A.WR, wq = (int)threadIdx.x >> 5;
    uint32_t* own = s_lat + kColor * BW;
    const uint32_t* oth = s_lat + (1 - kColor) * BW;
    // the neighbours' other-colour rows: band-1 of the CTA above, 0 of the one below
    const uint32_t* up_row = up_pl + (1 - kColor) * BW + (kRows - 1) * NS + NS - WR;
    const uint32_t* dn_row = dn_pl + (1 - kColor) * BW;
    if constexpr (kPre) {  // one strip per thread (NS == blockDim.x), planes drawn ahead
        smem_strip<kRows, kColor, kStats, true>(own, oth, up_row, dn_row, (int)threadIdx.x, WR, wr_shift, NS,
                                                band_lo, TM, TC, t3, t4, slot, A.rk, ctr1, s_tie[wq][0],
                                                s_tie[wq][1], s_tie[wq][2], sS, sB, Upre);
    } else {
        for (int s = (int)threadIdx.x; s < NS; s += (int)blockDim.x)
            smem_strip<kRows, kColor, kStats>(own, oth, up_row, dn_row, s, WR, wr_shift, NS, band_lo, TM, TC, t3,
                                              t4, slot, A.rk, ctr1, s_tie[wq][0], s_tie[wq][1], s_tie[wq][2], sS,
                                              sB);
    }
}

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// kPre: one strip per thread (NS == blockDim.x); the random planes of each
// pass are drawn ahead, off the critical path (smem_draws)
template <int kRows, int kThreads, bool kPre = false>
__global__ void __launch_bounds__(kThreads) cb_cluster_smem_kernel(ResidentArgs A) {
    extern __shared__ uint32_t s_lat[];  // [2][band * WR], band_word layout
    __shared__ uint32_t s_mask[19];      // TM[8], TC[8], t3, t4, slot
    __shared__ int s_part[2][2];         // rank 0: the lattice's (S, Bond), by sweep parity
    __shared__ uint32_t s_tie[kThreads / 32][3][kRows][32];
    cg::cluster_group cluster = cg::this_cluster();
    const int cs = (int)cluster.num_blocks(), q = (int)cluster.block_rank();
    const int row = (int)blockIdx.x / cs;  // the cluster's lattice (local index)
    const int L = A.L, WR = A.WR, W = A.W;
    const int band = L / cs, BW = band * WR, NS = band / kRows * WR, band_lo = q * band;
    const int wr_shift = (WR & (WR - 1)) == 0 ? __ffs(WR) - 1 : -1;
    const bool multi = A.world > 1;
    const int R = multi ? A.R_total : A.R;  // slots (pairs, swap streams, ring entries)
    uint32_t* const gl = A.packed + (int64_t)row * 2 * W;
    for (int c = 0; c < 2; ++c)
        for (int x = (int)threadIdx.x; x < BW; x += (int)blockDim.x) {
            const int rl = x / WR, k = x - rl * WR;
            s_lat[c * BW + band_word<kRows>(rl, k, WR, NS)] = gl[(int64_t)c * W + band_lo * WR + x];
        }
    if (threadIdx.x == 0) {
        const int k = A.r2s[A.buf][row];
        smem_set_slot(k, __ldg(A.thresh + k * 10 + 8), __ldg(A.thresh + k * 10 + 9), s_mask);
    }
    const uint32_t* up_pl = cluster.map_shared_rank(s_lat, (q + cs - 1) % cs);
    const uint32_t* dn_pl = cluster.map_shared_rank(s_lat, (q + 1) % cs);
    uint64_t* const ring = reinterpret_cast<uint64_t*>(A.slot_stats);  // kRing x R words
    cluster.sync();  // every band loaded before a neighbour reads its halo
    // (The cluster barrier is the cheapest separation of the colours measured:
    // release/acquire phase flags pushed into the neighbours' shared memory
    // cost ~2x more per phase.)
    int rounds = 0;
    // kPre: the next colour-0 pass's planes, for the lattice's slot (U0) and,
    // across a round, for the partner's slot too (U0x, taken if the swap is
    // accepted); the colour-1 pass's (U1)
    uint32_t U0[kRows][8], U0x[kRows][8], U1[kRows][8];
    if constexpr (kPre)
        smem_draws<kRows>((int)threadIdx.x, WR, wr_shift, band_lo, s_mask[18], A.rk, (uint32_t)(2 * A.first_sweep), U0);
    RunSchedule sx, sr;
    sx.init(A.swap_every, A.first_sweep + 1);
    sr.init(A.record_every, A.first_sweep + 1);
    for (int64_t t = A.first_sweep; t < A.first_sweep + A.n_sweeps; ++t, sx.step(), sr.step()) {
        const int64_t done = t + 1;
        const bool rec = sr.hit();
        const bool exch = sx.hit() && done < A.total_sweeps;
        const bool last = t + 1 == A.first_sweep + A.n_sweeps;
        const bool need_stats = rec || exch || last;
        const int par = (int)(t & 1);
        // The round's inputs that do not depend on the partner (its slot, swap
        // draw, betas and thresholds), loaded by thread 0 before the sweep so
        // that their latency overlaps it.
        int k = 0, other = -1, si = 0;
        int64_t round = 0;
        double u = 0.0, bi = 0.0, bj = 0.0;  // (nothing consumes them before the decision)
        uint32_t ot3 = 0, ot4 = 0;
        if (threadIdx.x == 0) {
            k = (int)s_mask[18];
            if (exch) {
                round = sx.index();
                const int first = (int)(round & 1), n_pairs = (R - first) / 2;
                if (k >= first && (k - first) / 2 < n_pairs) {
                    const int p = (k - first) / 2;
                    si = first + 2 * p;
                    other = k == si ? si + 1 : si;
                    u = A.u_table[(round - A.u_round0) * A.u_stride + p];
                    bi = A.betas[si];
                    bj = A.betas[si + 1];
                    ot3 = __ldg(A.thresh + other * 10 + 8);
                    ot4 = __ldg(A.thresh + other * 10 + 9);
                }
            }
            // rank 0 accumulates the lattice's (S, Bond): zeroed here, added to
            // after the colour-0 barrier; the other ranks last read this
            // parity's sums before the previous sweep's colour-0 barrier
            if (q == 0) {
                s_part[par][0] = 0;
                s_part[par][1] = 0;
            }
        }
        int* const part0 = cluster.map_shared_rank(&s_part[par][0], 0);
        int sS = 0, sB = 0;
        smem_pass<kRows, kThreads, 0, false, kPre>(A, s_lat, up_pl, dn_pl, BW, NS, band_lo, wr_shift, s_mask,
                                                   (uint32_t)(2 * t), s_tie, sS, sB, U0);
        if constexpr (kPre) {  // colour 1's planes while the cluster catches up
            const uint32_t slot = s_mask[18];
            cluster_arrive();
            smem_draws<kRows>((int)threadIdx.x, WR, wr_shift, band_lo, slot, A.rk, (uint32_t)(2 * t + 1), U1);
            cluster_wait();
        } else {
            cluster.sync();
        }
        if (need_stats) {
            smem_pass<kRows, kThreads, 1, true, kPre>(A, s_lat, up_pl, dn_pl, BW, NS, band_lo, wr_shift, s_mask,
                                                      (uint32_t)(2 * t + 1), s_tie, sS, sB, U1);
            sS = __reduce_add_sync(kFullMask, sS);
            sB = __reduce_add_sync(kFullMask, sB);
            if ((threadIdx.x & 31) == 0) {  // DSMEM atomics into rank 0's sums
                atomicAdd(part0, sS);
                atomicAdd(part0 + 1, sB);
            }
        } else {
            smem_pass<kRows, kThreads, 1, false, kPre>(A, s_lat, up_pl, dn_pl, BW, NS, band_lo, wr_shift, s_mask,
                                                       (uint32_t)(2 * t + 1), s_tie, sS, sB, U1);
        }
        // colour 1 done everywhere, rank 0's sums complete
        uint32_t cur = 0, alt = 0;
        if constexpr (kPre) {
            // the next colour 0's planes while the cluster catches up: for the
            // lattice's slot and, if it is paired in this sweep's round, for
            // the partner's (the round may hand the lattice that slot)
            cur = s_mask[18];  // (read before arriving: thread 0 may update it once the cluster has arrived)
            cluster_arrive();
            alt = cur;
            if (exch) {
                const int64_t rd = sx.index();
                const int first = (int)(rd & 1), n_pairs = (R - first) / 2;
                const int kc = (int)cur;
                if (kc >= first && (kc - first) / 2 < n_pairs) {
                    const int si0 = first + 2 * ((kc - first) / 2);
                    alt = (uint32_t)(kc == si0 ? si0 + 1 : si0);
                }
            }
            const uint32_t c0n = (uint32_t)(2 * t + 2);
            smem_draws<kRows>((int)threadIdx.x, WR, wr_shift, band_lo, cur, A.rk, c0n, U0);
            if (alt != cur) smem_draws<kRows>((int)threadIdx.x, WR, wr_shift, band_lo, alt, A.rk, c0n, U0x);
            cluster_wait();
        } else {
            cluster.sync();
        }
        if (!need_stats) continue;
        if (threadIdx.x == 0) {
            const int64_t S = part0[0], Bd = part0[1];
            if (q == 0) {
                if (exch) {  // first: the partner is waiting for it
                    const int64_t ro = (round & (kRing - 1)) * (int64_t)R;
                    const uint64_t mine = p2p_pack(S, Bd, round);
                    if (multi) {
                        for (int g = 0; g < A.world; ++g)
                            st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(A.pub_peer[g]) + ro + k, mine);
                    } else {
                        st_relaxed_u64(ring + ro + k, mine);
                    }
                }
                if (last) {
                    A.stats[2 * row] = S;
                    A.stats[2 * row + 1] = Bd;
                }
                if (rec) {  // by slot, before the round (executor.py order)
                    const int64_t col = sr.index();
                    A.obs_e[(int64_t)k * A.ncols + col] =
                        __dsub_rn(__dmul_rn(A.B, (double)S), __dmul_rn(A.J, (double)Bd));
                    A.obs_m[(int64_t)k * A.ncols + col] = __ddiv_rn((double)S, (double)A.L * A.L);
                }
            }
            if (other >= 0) {
                const uint64_t want = (uint64_t)((round & 0x7fff) | 0x8000);
                const uint64_t* src = ring + (round & (kRing - 1)) * (int64_t)R + other;
                uint64_t v = multi ? ld_relaxed_sys_u64(src) : ld_relaxed_u64(src);
                while ((v & 0xffffull) != want) {
                    __nanosleep(32);
                    v = multi ? ld_relaxed_sys_u64(src) : ld_relaxed_u64(src);
                }
                const int64_t So = p2p_field(v, 16), Bo = p2p_field(v, 40);
                const bool mine_i = k == si;
                const int64_t Si = mine_i ? S : So, Bi = mine_i ? Bd : Bo;
                const int64_t Sj = mine_i ? So : S, Bj = mine_i ? Bo : Bd;
                const double Ei = __dsub_rn(__dmul_rn(A.B, (double)Si), __dmul_rn(A.J, (double)Bi));
                const double Ej = __dsub_rn(__dmul_rn(A.B, (double)Sj), __dmul_rn(A.J, (double)Bj));
                bool near = false;
                const bool acc = swap_decide(__dsub_rn(bi, bj), Ei, Ej, u, near);
                if (mine_i && q == 0) {
                    if (acc) atomicAdd((unsigned long long*)&A.counters[0], 1ull);
                    if (near) atomicAdd((unsigned long long*)&A.counters[1], 1ull);
                }
                if (acc) smem_set_slot(other, ot3, ot4, s_mask);
            }
        }
        if (exch) ++rounds;
        __syncthreads();  // the next sweep reads s_mask
        if constexpr (kPre) {
            if (s_mask[18] != cur) {  // the swap was accepted: the partner slot's planes
#pragma unroll
                for (int rr = 0; rr < kRows; ++rr)
#pragma unroll
                    for (int p = 0; p < 8; ++p) U0[rr][p] = U0x[rr][p];
            }
        }
    }
    // the band back to global memory; the permutation where the grid-barrier
    // kernel would leave it (its buffer flips once per round)
    for (int c = 0; c < 2; ++c)
        for (int x = (int)threadIdx.x; x < BW; x += (int)blockDim.x) {
            const int rl = x / WR, k = x - rl * WR;
            gl[(int64_t)c * W + band_lo * WR + x] = s_lat[c * BW + band_word<kRows>(rl, k, WR, NS)];
        }
    if (q == 0 && threadIdx.x == 0) {
        const int fb = A.buf ^ (rounds & 1);
        const int k = (int)s_mask[18];
        A.r2s[fb][row] = k;
        A.s2r[fb][k] = A.row_lo + row;
    }
    cluster.sync();  // no CTA leaves while a neighbour may still read its shared memory
}


template <int kRows, int kThreads>
static int launch_smem_t(const ResidentArgs& a, int cs, cudaStream_t s) {
    const int band = a.L / cs;
    if (band % kRows != 0) return kNotApplicable;
    const int NS = band / kRows * a.WR;
    if (NS % 32 != 0) return kNotApplicable;  // whole warps walk their ties together
    const size_t smem = 2 * (size_t)band * a.WR * sizeof(uint32_t);
    // one strip per thread: the planes drawn ahead (kPre); PTMH_SMEM_PRE=0 turns it off
    const char* ep = getenv("PTMH_SMEM_PRE");
    const bool pre = NS <= kThreads && !(ep && ep[0] == '0');
    const void* fn = pre ? (const void*)cb_cluster_smem_kernel<kRows, kThreads, true>
                         : (const void*)cb_cluster_smem_kernel<kRows, kThreads, false>;
    if (cs > 8) PTMH_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (smem > 48 * 1024)
        PTMH_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int threads = std::min(kThreads, NS);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.R * cs));
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    // Without the cooperative attribute under Nsight Compute (which sets
    // NV_COMPUTE_PROFILER_PERFWORKS_DIR / NV_NSIGHT_INJECTION_PORT_BASE in the
    // target) or with PTMH_SMEM_NOCOOP=1: ncu fails cooperative cluster
    // launches with dynamic shared memory (LaunchFailed).  Every cluster is
    // still resident at once: the launcher checked that they all fit, and a
    // profiled kernel runs alone.
    const char* nc = getenv("PTMH_SMEM_NOCOOP");
    const bool profiled = getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") != nullptr ||
                          getenv("NV_NSIGHT_INJECTION_PORT_BASE") != nullptr;
    cfg.numAttrs = ((nc && nc[0] == '1') || profiled) ? 1 : 2;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return kNotApplicable;
    }
    const int cap = a.max_ctas > 0 ? a.max_ctas / cs : ncl;
    if (std::min(ncl, cap) < a.R) return kNotApplicable;  // every cluster must be resident
    if (a.swap_every > 0 && a.world == 1)
        PTMH_CUDA(cudaMemsetAsync(a.slot_stats, 0, (size_t)kRing * a.R * 8, s));
    void* kargs[] = {const_cast<ResidentArgs*>(&a)};
    const cudaError_t le = cudaLaunchKernelExC(&cfg, fn, kargs);
    if (le == cudaErrorCooperativeLaunchTooLarge) {
        // the occupancy query can admit a grid that the cooperative launch
        // then refuses (cluster placement): resident.cu's kernel instead
        cudaGetLastError();
        return kNotApplicable;
    }
    PTMH_CUDA(le);
    cb_set_last_launch(CbLaunchInfo{8, kRows, threads, cs, 0, a.R * cs});
    return PTMH_OK;
}

// Applies to ferro lattices with L % 64 == 0 and more than 64 words per
// colour (smaller ones are warp-owned in resident.cu), a swap-draw table
// (point-to-point rounds), and when every cluster fits on the GPU at once.
// Returns kNotApplicable (1) when the caller should use resident.cu.
int launch_cb_cluster_smem(const ResidentArgs& a, cudaStream_t s) {
    const char* e = getenv("PTMH_RESIDENT_SMEM");  // "0": off; "cs,rows,threads": that configuration
    if (e && e[0] == '0') return kNotApplicable;
    const char* ep = getenv("PTMH_RESIDENT_P2P");  // "0": grid-barrier rounds (resident.cu)
    if (ep && ep[0] == '0' && a.swap_every > 0) return kNotApplicable;
    if (!a.ferro || a.WR <= 0 || a.W <= 64 || (!a.u_table && a.swap_every > 0)) return kNotApplicable;
    if (a.L > 1024) return kNotApplicable;  // the round word's 24-bit (S, Bond) fields (rounds.cuh)
    int dev = 0, sms = 0;
    PTMH_CUDA(cudaGetDevice(&dev));
    PTMH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int cs = 0, rows = 2, threads = 256;
    if (e && e[0] != '\0') {
        if (sscanf(e, "%d,%d,%d", &cs, &rows, &threads) != 3) return kNotApplicable;
    } else {
        // clusters of cs CTAs: up to as many CTAs as SMs, at most 8 per
        // cluster, while the band still splits into whole warps of 2-row strips
        auto whole_warps = [&](int c) {
            const int band = a.L / c;
            return a.L % c == 0 && band % 2 == 0 && (band / 2 * a.WR) % 32 == 0;
        };
        cs = 1;
        while (cs < 8 && (int64_t)a.R * cs * 2 <= sms && whole_warps(cs * 2)) cs *= 2;
        // 1-row strips on 512 threads where that gives every thread exactly
        // one strip (the planes drawn ahead) on clusters of <= 2 CTAs: C2
        // 4.84 -> 4.75 us per sweep + round (512^2 x 16 on 8-CTA clusters of
        // 512-thread CTAs does not get its clusters placed)
        const char* e1 = getenv("PTMH_SMEM_ROWS1");
        if (!(e1 && e1[0] == '0') && cs <= 2 && (a.L / cs) * a.WR == 512) {
            rows = 1;
            threads = 512;
        }
    }
    if (cs < 1 || cs > 16 || a.L % cs != 0) return kNotApplicable;
    if (rows == 1 && threads == 256) return launch_smem_t<1, 256>(a, cs, s);
    if (rows == 1 && threads == 512) return launch_smem_t<1, 512>(a, cs, s);
    if (rows == 2 && threads == 128) return launch_smem_t<2, 128>(a, cs, s);
    if (rows == 2 && threads == 256) return launch_smem_t<2, 256>(a, cs, s);
    if (rows == 2 && threads == 512) return launch_smem_t<2, 512>(a, cs, s);
    if (rows == 4 && threads == 128) return launch_smem_t<4, 128>(a, cs, s);
    if (rows == 4 && threads == 256) return launch_smem_t<4, 256>(a, cs, s);
    return kNotApplicable;
}

}  // namespace ptmh

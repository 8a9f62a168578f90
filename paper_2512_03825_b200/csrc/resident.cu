// resident.cu -- persistent checkerboard PT run for small and many lattices.
//
// One cooperative launch runs many sweeps *and* the exchange rounds between
// them.  Each CTA owns whole lattices (lattice r -> CTA r % gridDim.x), so the
// two colour half-sweeps of a lattice only need __syncthreads, and its (S, Bond)
// come from a block reduction (no atomics).  The only grid-wide barrier is the
// one before an exchange round, when every lattice's energy must be final.
//
// Exchange without a second barrier: the owner of lattice r (slot k) decides
// the pair containing k itself -- both owners of a pair evaluate the same
// reference rule (kernels.py:116-148) on the same inputs (energies from stats,
// the swap draw at stream R+p, position = round), so they agree -- and writes
// r's new slot into the *other* buffer of the double-buffered permutation.
// Partner lookups read the current buffer, which nobody writes this round.
//
// The per-word update is the same arithmetic as checkerboard.cu (same chain,
// same random numbers, bit-exact with oracle/ptmh_oracle.c); ties are resolved
// in place by the owning lane.
#include <cooperative_groups.h>
#include <cstdlib>
#include <cuda_runtime.h>

#include "common.cuh"
#include "launchers.cuh"
#include "philox.cuh"
#include "rounds.cuh"
#include "strip.cuh"

namespace cg = cooperative_groups;

namespace ptmh {

// ResidentArgs is declared in launchers.cuh

__device__ __forceinline__ uint32_t resident_bit(const uint32_t* p, int h) {
    return (p[h >> 5] >> (h & 31)) & 1u;
}

// one colour-c word of a lattice: gather neighbour words, decide, store;
// returns nothing, adds the colour-1 (S, Bond) contributions when `stats`
// gather modes: rows of 64+ sites (L % 64 == 0), whole rows per word
// (L = 8, 16, 32: a word holds 64 / L rows of L/2 same-colour sites), any even L
enum { kGatherGeneric = 0, kGatherRows = 1, kGatherSegments = 2 };

template <int kMode, bool kFerro>
__device__ __forceinline__ void resident_word(const ResidentArgs& A, uint32_t* own, const uint32_t* oth,
                                              int w, int color, int slot, uint32_t ctr1, int& sumS,
                                              int& sumB, bool stats, const uint32_t* masks, int wr_shift) {
    const int L = A.L;
    uint32_t S = own[w], n1, n2, n3, n4, valid;
    if (kMode == kGatherRows) {
        const int WR = A.WR;
        const int i = wr_shift >= 0 ? (w >> wr_shift) : w / WR, k = w - i * WR;
        const int iu = (i == 0) ? L - 1 : i - 1, id = (i == L - 1) ? 0 : i + 1;
        const uint32_t mid = oth[w];
        n1 = oth[iu * WR + k];
        n2 = oth[id * WR + k];
        n3 = mid;
        if (((i + color) & 1) == 0) {
            n4 = __funnelshift_l(oth[i * WR + (k == 0 ? WR - 1 : k - 1)], mid, 1);
        } else {
            n4 = __funnelshift_r(mid, oth[i * WR + (k == WR - 1 ? 0 : k + 1)], 1);
        }
        valid = 0xffffffffu;
    } else if (kMode == kGatherSegments) {
        // word w = rows w*q .. w*q+q-1 of this colour, q = 64 / L, seg = L / 2
        // sites each; q is even, so segment s has row parity s & 1
        const int seg = L >> 1, W = A.W;
        const uint32_t mid = oth[w];
        const uint32_t prev = oth[w == 0 ? W - 1 : w - 1], next = oth[w == W - 1 ? 0 : w + 1];
        n1 = __funnelshift_l(prev, mid, seg);       // row above: previous segment
        n2 = __funnelshift_r(mid, next, seg);       // row below: next segment
        n3 = mid;
        const uint32_t lo_bits = A.seg_lo, hi_bits = lo_bits << (seg - 1);  // bit 0 / top bit of each segment
        const uint32_t rot_l = ((mid << 1) & ~lo_bits) | ((mid >> (seg - 1)) & lo_bits);  // site m-1
        const uint32_t rot_r = ((mid >> 1) & ~hi_bits) | ((mid << (seg - 1)) & hi_bits);  // site m+1
        const uint32_t even = color ? ~A.seg_even : A.seg_even;  // segments with (row + colour) even
        n4 = (rot_l & even) | (rot_r & ~even);
        valid = 0xffffffffu;
    } else {
        const int Lh = L / 2, H = L * Lh;
        n1 = n2 = n3 = n4 = valid = 0;
        for (int b = 0; b < 32; ++b) {
            const int h = w * 32 + b;
            if (h >= H) break;
            valid |= 1u << b;
            const int i = h / Lh, m = h - i * Lh;
            const int j = 2 * m + ((i + color) & 1);
            const int iu = (i == 0) ? L - 1 : i - 1, id = (i == L - 1) ? 0 : i + 1;
            const int jl = (j == 0) ? L - 1 : j - 1, jr = (j == L - 1) ? 0 : j + 1;
            n1 |= resident_bit(oth, iu * Lh + (j >> 1)) << b;
            n2 |= resident_bit(oth, id * Lh + (j >> 1)) << b;
            n3 |= resident_bit(oth, i * Lh + (jl >> 1)) << b;
            n4 |= resident_bit(oth, i * Lh + (jr >> 1)) << b;
        }
    }
    const uint32_t a = ~(S ^ n1), b = ~(S ^ n2), c = ~(S ^ n3), d = ~(S ^ n4);
    const uint32_t s1 = a ^ b, c1 = a & b, s2 = c ^ d, c2 = c & d;
    const uint32_t k0 = s1 ^ s2, c3 = s1 & s2;
    const uint32_t k1 = c1 ^ c2 ^ c3, k2 = c1 & c2;
    const uint32_t* thr = A.thresh + slot * 10;
    uint32_t acc;
    if (kFerro) {
        // J > 0, B = 0: k <= 1 always, k = 2 with probability 1/2, k = 3, 4 thresholds
        const uint32_t K4 = k2, upm = ((k1 & k0) | k2) & valid, K2 = k1 & ~k0 & valid;
        const uint32_t t3 = masks[16], t4 = masks[17];  // per-lattice, in shared memory
        acc = ~(k1 | k2) & valid;
        const uint4 r0 = philox4x32_10(make_uint4(2u * (uint32_t)w, ctr1, (uint32_t)slot, 0u), A.rk);
        const uint4 r1 = philox4x32_10(make_uint4(2u * (uint32_t)w + 1u, ctr1, (uint32_t)slot, 0u), A.rk);
        const uint32_t U[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
        acc |= K2 & ~U[0];
        uint32_t bor = 0, eq = upm;  // borrow of u - t (LSB first) + ties
#pragma unroll
        for (int p = 7; p >= 0; --p) {
            // threshold plane: t4's bit where K4, else t3's, as one IMAD
            // (checkerboard.cu, ferro_strip)
            const uint32_t Tm = K4 * masks[p] + masks[8 + p];
            bor = (~U[p] & Tm) | (~U[p] & bor) | (Tm & bor);
            eq &= ~(U[p] ^ Tm);
        }
        acc |= bor & upm;
        while (eq) {
            const int bit = __ffs(eq) - 1;
            eq &= eq - 1;
            const uint32_t t24 = (((K4 >> bit) & 1u) ? t4 : t3) & 0x00ffffffu;
            const uint4 r2 =
                philox4x32_10(make_uint4((uint32_t)w * 32u + (uint32_t)bit, ctr1, (uint32_t)slot, 1u), A.rk);
            if ((r2.x >> 8) < t24) acc |= 1u << bit;
        }
    } else {
        uint32_t K[5];
        K[4] = k2;
        K[3] = k1 & k0;
        K[2] = k1 & ~k0;
        K[1] = k0 & ~k1;
        K[0] = ~(k0 | k1 | k2);
        uint32_t M[10], T[10], up = 0;
        const int nq = A.n_up;
#pragma unroll
        for (int q = 0; q < 10; ++q) {
            if (q < nq) {
                const uint32_t sf = A.up_sf[q] == 0 ? 0xffffffffu : (A.up_sf[q] == 1 ? S : ~S);
                M[q] = K[A.up_k[q]] & sf & valid;
                T[q] = __ldg(thr + A.up_cls[q]);
                up |= M[q];
            } else {
                M[q] = 0;
                T[q] = 0;
            }
        }
        acc = valid & ~up;
        if (up) {
            const uint4 r0 = philox4x32_10(make_uint4(2u * (uint32_t)w, ctr1, (uint32_t)slot, 0u), A.rk);
            const uint4 r1 = philox4x32_10(make_uint4(2u * (uint32_t)w + 1u, ctr1, (uint32_t)slot, 0u), A.rk);
            const uint32_t U[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
            uint32_t lt = 0, eq = up;
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                uint32_t Tm = 0;
#pragma unroll
                for (int q = 0; q < 10; ++q)
                    if (q < nq) Tm |= M[q] & (0u - ((T[q] >> (31 - p)) & 1u));
                lt |= eq & ~U[p] & Tm;
                eq &= ~(U[p] ^ Tm);
            }
            acc |= lt;
            while (eq) {
                const int bit = __ffs(eq) - 1;
                eq &= eq - 1;
                uint32_t t24 = 0;
#pragma unroll
                for (int q = 0; q < 10; ++q)
                    if (q < nq && ((M[q] >> bit) & 1u)) t24 = T[q] & 0x00ffffffu;
                const uint4 r2 = philox4x32_10(
                    make_uint4((uint32_t)w * 32u + (uint32_t)bit, ctr1, (uint32_t)slot, 1u), A.rk);
                if ((r2.x >> 8) < t24) acc |= 1u << bit;
            }
        }
    }
    const uint32_t Sn = S ^ acc;
    if (acc) own[w] = Sn;
    if (stats) {  // colour-1 pass: absolute (S, Bond) of the new configuration
        const int kk = __popc((a ^ acc) & valid) + __popc((b ^ acc) & valid) + __popc((c ^ acc) & valid) +
                       __popc((d ^ acc) & valid);
        const int nv = __popc(valid);
        sumB += 2 * kk - 4 * nv;
        sumS += 2 * (__popc(Sn & valid) + __popc(oth[w] & valid)) - 2 * nv;
    }
}

constexpr int kMaxLatPerBlock = 64;

// lattice li of this block now holds `slot`: cache its slot and (ferro) the
// threshold-plane select coefficients in shared memory
template <bool kFerro>
__device__ __forceinline__ void resident_set_slot(const ResidentArgs& A, int li, int slot, int* s_slot,
                                                  uint32_t (*s_mask)[19]) {
    s_slot[li] = slot;
    if (kFerro) {
        const uint32_t t3 = __ldg(A.thresh + slot * 10 + 8), t4 = __ldg(A.thresh + slot * 10 + 9);
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            const uint32_t ta = (t3 >> (31 - p)) & 1u, tb = (t4 >> (31 - p)) & 1u;
            s_mask[li][p] = tb - ta;     // TM: Tm = K4 * TM + TC
            s_mask[li][8 + p] = 0u - ta;  // TC
        }
        s_mask[li][16] = t3;
        s_mask[li][17] = t4;
        s_mask[li][18] = (uint32_t)slot;
    }
}

// Block b owns the contiguous lattices [lo, hi) and sweeps them together:
// work items (lattice, word) are spread over all threads, __syncthreads
// separates the colours, per-lattice (S, Bond) accumulate in shared memory.
// Slots live in shared memory for the whole launch: only the owner changes
// them, after an exchange round.
//
// kCl: a thread-block CLUSTER owns the lattices instead (when there are fewer
// lattices than SMs, e.g. C2's 64 lattices of 256^2): its CTAs split the
// (lattice, word) items, the cluster barrier separates the colours, and the
// per-lattice (S, Bond) partial sums go to rank 0's shared memory through
// DSMEM atomics.  Every CTA keeps its own copy of the slots and masks and
// decides the exchange for its cluster's lattices redundantly (same inputs,
// same rule); rank 0 alone writes the outputs.
template <int kMode, bool kFerro, int kThreads, bool kCl>
__global__ void __launch_bounds__(kThreads, kThreads <= 256 ? 2 : 1) cb_resident_kernel(ResidentArgs A) {
    __shared__ int s_slot[kMaxLatPerBlock];
    __shared__ int s_S[kMaxLatPerBlock], s_B[kMaxLatPerBlock];
    // point-to-point rounds on clusters: (S, Bond) accumulate in rank 0's
    // buffer [t & 1], zeroed two sweeps after it was last read
    __shared__ int s_Sc[kCl ? 2 : 1][kCl ? kMaxLatPerBlock : 1], s_Bc[kCl ? 2 : 1][kCl ? kMaxLatPerBlock : 1];
    __shared__ double s_u[kMaxLatPerBlock];
    __shared__ double s_bd[kMaxLatPerBlock];       // beta_i - beta_j of the slot's pair (this round)
    __shared__ uint32_t s_pt[kMaxLatPerBlock][2];  // thresholds t3, t4 of the partner slot (ferro)
    __shared__ uint32_t s_mask[kFerro ? kMaxLatPerBlock : 1][19];  // TM[8], TC[8], t3, t4, slot
    // warp-owned 64^2 ferro lattices run the sweep kernels' strip code (2-row
    // strips, one per lane): its tie scratch, per warp
    constexpr bool kStrip = kFerro && kMode == kGatherRows && !kCl;
    __shared__ uint32_t s_tie[kStrip ? kThreads / 32 : 1][3][2][32];
    // Next round's swap draws, for runs of <= 32 pairs: a warp the exchange
    // decisions leave idle computes them while the decisions run, so the
    // next publish does not wait on a Philox4x64 chain (C1: the draw was 12 %
    // of a sweep + round).  s_pre_round: the round they belong to, or -1.
    __shared__ double s_unext[32];
    __shared__ long long s_pre_round;
    cg::cluster_group cluster = cg::this_cluster();
    const int cs = kCl ? (int)cluster.num_blocks() : 1;
    const int crank = kCl ? (int)cluster.block_rank() : 0;
    const int cid = (int)blockIdx.x / cs, ncl = (int)gridDim.x / cs;
    int* s_S0 = kCl ? cluster.map_shared_rank(s_S, 0) : s_S;  // rank 0 accumulates
    int* s_B0 = kCl ? cluster.map_shared_rank(s_B, 0) : s_B;
    const bool owner = crank == 0;
    const int wr_shift = (A.WR > 0 && (A.WR & (A.WR - 1)) == 0) ? __ffs(A.WR) - 1 : -1;
    const int W = A.W;
    const int R = A.world > 1 ? A.R_total : A.R;  // slots (pairs, swap streams, pub indices)
    const int lo = (int)((int64_t)A.R * cid / ncl);  // this CTA's (local) lattices
    const int hi = (int)((int64_t)A.R * (cid + 1) / ncl);
    const int nl = hi - lo;
    // this CTA's slice [ib, ib + items) of the cluster's (lattice, word) items
    const int ib = (int)((int64_t)nl * W * crank / cs);
    const int items = (int)((int64_t)nl * W * (crank + 1) / cs) - ib;
    const int items_pad = (items + 31) & ~31;  // whole warps iterate together (warp-reduced stats)
    // (li, w) of this thread's first item and the per-iteration step
    const int li_0 = (ib + (int)threadIdx.x) / W, w_0 = ib + (int)threadIdx.x - li_0 * W;
    const int step_l = (int)blockDim.x / W, step_w = (int)blockDim.x - step_l * W;
    int buf = A.buf;
    for (int i = threadIdx.x; i < nl; i += blockDim.x) {
        resident_set_slot<kFerro>(A, i, A.r2s[buf][lo + i], s_slot, s_mask);
        s_S[i] = 0;
        s_B[i] = 0;
    }
    if (threadIdx.x == 0) s_pre_round = -1;
    const int pre_warp = (nl + 31) / 32;  // first warp without an exchange decision
    const bool pre = R / 2 <= 32 && (int)blockDim.x >= 32 * (pre_warp + 1);
    if (kCl)
        cluster.sync();
    else
        __syncthreads();
    const bool p2p = kCl && A.p2p;
    int p2p_rounds = 0;
    for (int64_t t = A.first_sweep; t < A.first_sweep + A.n_sweeps; ++t) {
        const int64_t done = t + 1;
        const bool rec = A.record_every > 0 && done % A.record_every == 0;
        const bool exch = A.swap_every > 0 && done % A.swap_every == 0 && done < A.total_sweeps;
        const bool need_stats = rec || exch || t + 1 == A.first_sweep + A.n_sweeps;
        if (p2p) {  // this sweep's accumulators (the colour-0 barrier orders this before the adds)
            s_S0 = cluster.map_shared_rank(&s_Sc[t & 1][0], 0);
            s_B0 = cluster.map_shared_rank(&s_Bc[t & 1][0], 0);
            if (owner)
                for (int i = threadIdx.x; i < nl; i += blockDim.x) {
                    s_Sc[t & 1][i] = 0;
                    s_Bc[t & 1][i] = 0;
                }
        }
        if (!kCl && A.warp_lat) {
            // warp-owned lattices: warp q sweeps lattices q, q + nwarps, ...
            // whole (both colours, lanes striding over the words), so the
            // colours only need __syncwarp and the warps never wait for each
            // other between exchange rounds
            const int lane = threadIdx.x & 31, nwarps = (int)blockDim.x >> 5;
            for (int color = 0; color < 2; ++color) {
                const uint32_t ctr1 = (uint32_t)(2 * t + color);
                const bool st = color == 1 && need_stats;
                for (int li = (int)threadIdx.x >> 5; li < nl; li += nwarps) {
                    uint32_t* c0 = A.packed + (int64_t)(lo + li) * 2 * W;
                    uint32_t* own = color ? c0 + W : c0;
                    const uint32_t* oth = color ? c0 : c0 + W;
                    int sS = 0, sB = 0;
                    if (kStrip && A.strip) {
                        // L = 64: lane = a 2-row strip (rolling window, one tie walk per strip)
                        const int wq = (int)threadIdx.x >> 5;
                        uint32_t(&tm)[2][32] = s_tie[kStrip ? wq : 0][0];
                        uint32_t(&tk)[2][32] = s_tie[kStrip ? wq : 0][1];
                        uint32_t(&tn)[2][32] = s_tie[kStrip ? wq : 0][2];
                        if (color == 0)
                            ferro_strip<2, 0, false, false>(A.packed, A.L, 1, W, nullptr, A.thresh, A.rk, ctr1,
                                                            nullptr, 4u, true, lo + li, lane, tm, tk, tn, sS, sB,
                                                            0, s_mask[li]);
                        else if (st)
                            ferro_strip<2, 1, true, false>(A.packed, A.L, 1, W, nullptr, A.thresh, A.rk, ctr1,
                                                           nullptr, 4u, true, lo + li, lane, tm, tk, tn, sS, sB,
                                                           0, s_mask[li]);
                        else
                            ferro_strip<2, 1, false, false>(A.packed, A.L, 1, W, nullptr, A.thresh, A.rk, ctr1,
                                                            nullptr, 4u, true, lo + li, lane, tm, tk, tn, sS, sB,
                                                            0, s_mask[li]);
                    } else {
                        for (int w = lane; w < W; w += 32)
                            resident_word<kMode, kFerro>(A, own, oth, w, color, s_slot[li], ctr1, sS, sB, st,
                                                         kFerro ? s_mask[li] : nullptr, wr_shift);
                    }
                    if (st) {
                        for (int o = 16; o > 0; o >>= 1) {
                            sS += __shfl_down_sync(0xffffffffu, sS, o);
                            sB += __shfl_down_sync(0xffffffffu, sB, o);
                        }
                        if (lane == 0) {
                            s_S[li] += sS;
                            s_B[li] += sB;
                        }
                    }
                }
                __syncwarp();
            }
            if (need_stats) __syncthreads();  // every lattice's stats before the publish
        } else
        for (int color = 0; color < 2; ++color) {
            const uint32_t ctr1 = (uint32_t)(2 * t + color);
            const bool st = color == 1 && need_stats;
            int li_c = li_0, w_c = w_0;
            for (int it = threadIdx.x; it < items_pad; it += blockDim.x) {
                const bool on = it < items;
                const int li = on ? li_c : 0, w = on ? w_c : 0;
                li_c += step_l;
                w_c += step_w;
                if (w_c >= W) {
                    w_c -= W;
                    ++li_c;
                }
                int sS = 0, sB = 0;
                if (on) {
                    uint32_t* c0 = A.packed + (int64_t)(lo + li) * 2 * W;
                    uint32_t* own = color ? c0 + W : c0;
                    const uint32_t* oth = color ? c0 : c0 + W;
                    resident_word<kMode, kFerro>(A, own, oth, w, color, s_slot[li], ctr1, sS, sB, st,
                                                 kFerro ? s_mask[li] : nullptr, wr_shift);
                }
                if (st) {
                    const int li0 = __shfl_sync(0xffffffffu, li, 0);
                    if (__all_sync(0xffffffffu, li == li0 || !on)) {  // one lattice: one atomic
                        for (int o = 16; o > 0; o >>= 1) {
                            sS += __shfl_down_sync(0xffffffffu, sS, o);
                            sB += __shfl_down_sync(0xffffffffu, sB, o);
                        }
                        if ((threadIdx.x & 31) == 0) {
                            atomicAdd(&s_S0[li0], sS);
                            atomicAdd(&s_B0[li0], sB);
                        }
                    } else if (on) {
                        atomicAdd(&s_S0[li], sS);
                        atomicAdd(&s_B0[li], sB);
                    }
                }
            }
            if (kCl)
                cluster.sync();
            else
                __syncthreads();
        }
        if (!need_stats) continue;
        if (p2p) {
            // Point-to-point round (cb_resident_p2p_kernel's scheme for
            // cluster-owned lattices): rank 0 publishes each lattice's round
            // word; every CTA of the cluster polls the partner slot's word and
            // decides the pair redundantly (same inputs, same rule), so only
            // the partner is waited for, not the grid.
            const int64_t round = exch ? done / A.swap_every - 1 : 0;
            const int first = (int)(round % 2);
            const int n_pairs = (R - first) / 2;
            uint64_t* ring = reinterpret_cast<uint64_t*>(A.slot_stats) + (round % kRing) * (int64_t)R;
            for (int i = threadIdx.x; i < nl; i += blockDim.x) {
                const int64_t S = s_S0[i], Bd = s_B0[i];  // rank 0's sums (complete after the colour-1 barrier)
                const int k = s_slot[i];
                if (!owner) continue;
                if (t + 1 == A.first_sweep + A.n_sweeps) {
                    A.stats[2 * (lo + i)] = S;
                    A.stats[2 * (lo + i) + 1] = Bd;
                }
                if (rec) {
                    const int64_t col = done / A.record_every - 1;
                    A.obs_e[(int64_t)k * A.ncols + col] =
                        __dsub_rn(__dmul_rn(A.B, (double)S), __dmul_rn(A.J, (double)Bd));
                    A.obs_m[(int64_t)k * A.ncols + col] = __ddiv_rn((double)S, (double)A.L * A.L);
                }
                if (exch) st_relaxed_u64(ring + k, p2p_pack(S, Bd, round));
            }
            if (!exch) continue;
            ++p2p_rounds;
            for (int i = threadIdx.x; i < nl; i += blockDim.x) {
                const int k = s_slot[i];
                if (k < first || (k - first) / 2 >= n_pairs) continue;
                const int p = (k - first) / 2, si = first + 2 * p, sj = si + 1, other = k == si ? sj : si;
                const double u = A.u_table[(round - A.u_round0) * A.u_stride + p];
                const double bd = __dsub_rn(A.betas[si], A.betas[sj]);
                const uint32_t ot3 = kFerro ? __ldg(A.thresh + other * 10 + 8) : 0u;
                const uint32_t ot4 = kFerro ? __ldg(A.thresh + other * 10 + 9) : 0u;
                const int64_t S = s_S0[i], Bd = s_B0[i];
                const uint64_t want = (uint64_t)((round & 0x7fff) | 0x8000);
                uint64_t v = ld_relaxed_u64(ring + other);
                while ((v & 0xffffull) != want) {
                    __nanosleep(64);
                    v = ld_relaxed_u64(ring + other);
                }
                const int64_t So = p2p_field(v, 16), Bo = p2p_field(v, 40);
                const double Ei = __dsub_rn(__dmul_rn(A.B, (double)(k == si ? S : So)),
                                            __dmul_rn(A.J, (double)(k == si ? Bd : Bo)));
                const double Ej = __dsub_rn(__dmul_rn(A.B, (double)(k == si ? So : S)),
                                            __dmul_rn(A.J, (double)(k == si ? Bo : Bd)));
                bool near = false;
                const bool acc = swap_decide(bd, Ei, Ej, u, near);
                if (k == si && owner) {
                    if (acc) atomicAdd((unsigned long long*)&A.counters[0], 1ull);
                    if (near) atomicAdd((unsigned long long*)&A.counters[1], 1ull);
                }
                if (acc) {
                    s_slot[i] = other;
                    if (kFerro) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const uint32_t ta = (ot3 >> (31 - q)) & 1u, tb = (ot4 >> (31 - q)) & 1u;
                            s_mask[i][q] = tb - ta;
                            s_mask[i][8 + q] = 0u - ta;
                        }
                        s_mask[i][16] = ot3;
                        s_mask[i][17] = ot4;
                        s_mask[i][18] = (uint32_t)other;
                    }
                }
            }
            __syncthreads();  // next sweep reads s_slot / s_mask
            continue;
        }
        // publish (S, Bond); zero the accumulators for the next stats sweep
        // (the colour-0 barrier separates this from the next accumulation)
        const int64_t round = exch ? done / A.swap_every - 1 : 0;
        const int first = (int)(round % 2);
        const int n_pairs = (R - first) / 2;
        int64_t* pub = A.slot_stats + (round & 1) * 2 * (int64_t)R;
        for (int i = threadIdx.x; i < nl; i += blockDim.x) {
            const int k = s_slot[i];
            if (exch && k >= first && (k - first) / 2 < n_pairs) {
                // everything of the round that does not need the partner's
                // energy, before the barrier: the swap draw (stream R+p,
                // position = round), the pair's beta difference and the
                // partner slot's thresholds (their loads overlap the draw)
                const int pi = (k - first) / 2, si = first + 2 * pi, sj = si + 1;
                const double bi = A.betas[si], bj = A.betas[sj];
                const int other = (k == si) ? sj : si;
                const uint32_t t3 = kFerro ? __ldg(A.thresh + other * 10 + 8) : 0u;
                const uint32_t t4 = kFerro ? __ldg(A.thresh + other * 10 + 9) : 0u;
                s_u[i] = s_pre_round == round ? s_unext[pi]
                                               : stream_uniform(A.seed, (uint64_t)(R + pi), (uint64_t)round);
                s_bd[i] = __dsub_rn(bi, bj);
                s_pt[i][0] = t3;
                s_pt[i][1] = t4;
            } else if (exch) {
                s_u[i] = 0.0;
            }
            if (!owner) continue;
            const long long S = s_S[i], Bd = s_B[i];
            s_S[i] = 0;
            s_B[i] = 0;
            A.stats[2 * (lo + i)] = S;
            A.stats[2 * (lo + i) + 1] = Bd;
            if (rec) {  // by slot, before the round (executor.py order)
                const int64_t col = done / A.record_every - 1;
                A.obs_e[(int64_t)k * A.ncols + col] = __dsub_rn(__dmul_rn(A.B, (double)S), __dmul_rn(A.J, (double)Bd));
                A.obs_m[(int64_t)k * A.ncols + col] = __ddiv_rn((double)S, (double)A.L * A.L);
            }
            if (exch) {
                // the exchange reads (S, Bond) by slot: one load per partner
                pub[2 * k] = S;
                pub[2 * k + 1] = Bd;
                for (int g = 0; g < A.world; ++g) {  // sharded: every other rank's copy (NVLink peer stores)
                    if (g == A.rank) continue;
                    int64_t* pg = A.pub_peer[g] + (round & 1) * 2 * (int64_t)R;
                    pg[2 * k] = S;
                    pg[2 * k + 1] = Bd;
                }
            }
        }
        if (!exch) {
            if (!kCl && A.warp_lat) __syncthreads();  // the publish zeroed s_S before the next accumulation
            continue;
        }
        // every lattice's (S, Bond) is published.  (A point-to-point flag
        // scheme without this barrier was measured slower: DESIGN.md 5.)
        if (A.world > 1) {
            // every rank's (S, Bond) is published here when all ranks' flags
            // for this round arrived: publishers fence at system scope, the
            // grid barrier collects them, one thread signals every rank and
            // waits for every rank, a second grid barrier releases the CTAs
            __threadfence_system();
            cg::this_grid().sync();
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                const uint32_t want = (uint32_t)(round + 1);
                for (int g = 0; g < A.world; ++g)
                    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(A.flag_peer[g] + A.rank), "r"(want)
                                 : "memory");
                for (int g = 0; g < A.world; ++g) {
                    uint32_t v;
                    do {
                        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(A.flag_peer[A.rank] + g)
                                     : "memory");
                    } while ((int32_t)(v - want) < 0);
                }
            }
            cg::this_grid().sync();
        } else if (gridDim.x == 1) {
            __syncthreads();  // one CTA owns every lattice: the round needs no grid barrier
        } else {
            cg::this_grid().sync();
        }
        // ---- exchange round: the owner of lattice r decides the pair of its slot
        if (pre && ((int)threadIdx.x >> 5) == pre_warp) {  // (s_u of this round is read: the next is safe)
            const int lane = threadIdx.x & 31, nf = (int)((round + 1) % 2), np = (R - nf) / 2;
            if (lane < np) s_unext[lane] = stream_uniform(A.seed, (uint64_t)(R + lane), (uint64_t)(round + 1));
            if (lane == 0) s_pre_round = round + 1;
        }
        for (int li = threadIdx.x; li < nl; li += blockDim.x) {
            const int r = lo + li;
            const int k = s_slot[li];
            int nk = k;
            if (k >= first && (k - first) / 2 < n_pairs) {
                const int p = (k - first) / 2;
                const int i = first + 2 * p, j = i + 1;
                const double Ei = __dsub_rn(__dmul_rn(A.B, (double)pub[2 * i]), __dmul_rn(A.J, (double)pub[2 * i + 1]));
                const double Ej = __dsub_rn(__dmul_rn(A.B, (double)pub[2 * j]), __dmul_rn(A.J, (double)pub[2 * j + 1]));
                bool near = false;
                const bool acc = swap_decide(s_bd[li], Ei, Ej, s_u[li], near);
                if (acc) nk = (k == i) ? j : i;
                if (k == i && owner) {
                    if (acc) atomicAdd((unsigned long long*)&A.counters[0], 1ull);
                    if (near) atomicAdd((unsigned long long*)&A.counters[1], 1ull);
                }
            }
            // the permutation is an output only: nothing in the launch reads it back
            if (owner) {
                A.r2s[buf ^ 1][r] = nk;
                A.s2r[buf ^ 1][nk] = A.row_lo + r;  // sharded: only the slots held here
            }
            if (nk != k) {
                s_slot[li] = nk;
                if (kFerro) {  // resident_set_slot with the prefetched thresholds
                    const uint32_t t3 = s_pt[li][0], t4 = s_pt[li][1];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const uint32_t ta = (t3 >> (31 - q)) & 1u, tb = (t4 >> (31 - q)) & 1u;
                        s_mask[li][q] = tb - ta;
                        s_mask[li][8 + q] = 0u - ta;
                    }
                    s_mask[li][16] = t3;
                    s_mask[li][17] = t4;
                    s_mask[li][18] = (uint32_t)nk;
                }
            }
        }
        buf ^= 1;
        __syncthreads();  // next sweep reads s_slot / s_mask
    }
    if (p2p && owner) {  // the final mapping, where the grid-barrier rounds would leave it
        const int fb = A.buf ^ (p2p_rounds & 1);
        for (int i = threadIdx.x; i < nl; i += blockDim.x) {
            A.r2s[fb][lo + i] = s_slot[i];
            A.s2r[fb][s_slot[i]] = A.row_lo + lo + i;
        }
    }
}

// ------------------------------------------- point-to-point exchange rounds --
// The same run as cb_resident_kernel for warp-owned lattices on one GPU, with
// the exchange rounds decided pairwise instead of behind a grid barrier.  At
// a round the lattice's warp publishes its (S, Bond) for its slot k as ONE
// 64-bit word -- (S, Bond, round stamp) packed, so the value and its flag
// arrive together and no fence is needed -- into a 4-deep ring indexed by
// round, then polls the partner slot's word until it carries this round's
// stamp and decides the pair with the reference rule (both sides compute the
// same decision).  A warp therefore waits only for its partner, never for
// the slowest lattice of the grid, and while it waits the SM runs the other
// lattices' sweeps.
//
// Deadlock-free: every CTA is resident (cooperative launch), each warp owns
// one lattice, and the round-r publish of every slot depends only on round
// r-1 decisions, which depend on round r-1 publishes (induction on r).
// The ring is safe at depth 3: the next write to entry (r mod D, k) happens
// at round r+D, after its writer passed round r+D-1, which (chasing the
// pairings of rounds r+1 .. r+2, which alternate between the two neighbours)
// happens after the round-r reader of entry k decided; depth 4 is used.
// Stamps carry a valid bit, and the launcher zeroes the ring first, so an
// entry left by an earlier launch never matches.
// The swap draws (stream R+p, position = round; rng.py:113-116) come from a
// table the launcher fills before the launch (swap_draws_kernel): a
// Philox4x64-10 chain per round and lattice stays off the warps' path.
__global__ void swap_draws_kernel(uint64_t seed, int64_t R, int64_t round0, int64_t n_rounds, int64_t stride,
                                  double* __restrict__ out) {
    const int64_t n = n_rounds * stride;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / stride, p = t - r * stride;
        out[t] = stream_uniform(seed, (uint64_t)(R + p), (uint64_t)(round0 + r));
    }
}

template <int kMode, bool kFerro, int kThreads>
__global__ void __launch_bounds__(kThreads) cb_resident_p2p_kernel(ResidentArgs A) {
    constexpr int kWarps = kThreads / 32;
    __shared__ uint32_t s_mask[kWarps][19];  // the warp's lattice: TM[8], TC[8], t3, t4, slot
    __shared__ int s_slot[kWarps];
    constexpr bool kStrip = kFerro && kMode == kGatherRows;
    __shared__ uint32_t s_tie[kStrip ? kWarps : 1][3][2][32];
    const int lane = threadIdx.x & 31, wq = (int)threadIdx.x >> 5;
    const int W = A.W;
    // sharded (world > 1): this rank's A.R lattices, slots / pairs over R_total;
    // every lattice publishes into every rank's ring (NVLink peer stores) and
    // polls its own rank's ring
    const bool multi = A.world > 1;
    const int R = multi ? A.R_total : A.R;
    const int lo = (int)((int64_t)A.R * blockIdx.x / gridDim.x);
    const int hi = (int)((int64_t)A.R * (blockIdx.x + 1) / gridDim.x);
    if (wq >= hi - lo) return;  // no block-wide barrier below: spare warps leave
    const int row = lo + wq;
    const int wr_shift = (A.WR > 0 && (A.WR & (A.WR - 1)) == 0) ? __ffs(A.WR) - 1 : -1;
    uint32_t* const c0 = A.packed + (int64_t)row * 2 * W;
    uint64_t* const ring = reinterpret_cast<uint64_t*>(A.slot_stats);  // kRing x R words
    if (lane == 0) resident_set_slot<kFerro>(A, wq, A.r2s[A.buf][row], s_slot, s_mask);
    __syncwarp();
    int k = s_slot[wq];
    int rounds = 0;
    for (int64_t t = A.first_sweep; t < A.first_sweep + A.n_sweeps; ++t) {
        const int64_t done = t + 1;
        const bool rec = A.record_every > 0 && done % A.record_every == 0;
        const bool exch = A.swap_every > 0 && done % A.swap_every == 0 && done < A.total_sweeps;
        const bool last = t + 1 == A.first_sweep + A.n_sweeps;
        const bool need_stats = rec || exch || last;
        int sS = 0, sB = 0;
        for (int color = 0; color < 2; ++color) {
            const uint32_t ctr1 = (uint32_t)(2 * t + color);
            const bool st = color == 1 && need_stats;
            uint32_t* own = color ? c0 + W : c0;
            const uint32_t* oth = color ? c0 : c0 + W;
            if (kStrip && A.strip) {
                uint32_t(&tm)[2][32] = s_tie[kStrip ? wq : 0][0];
                uint32_t(&tk)[2][32] = s_tie[kStrip ? wq : 0][1];
                uint32_t(&tn)[2][32] = s_tie[kStrip ? wq : 0][2];
                if (color == 0)
                    ferro_strip<2, 0, false, false>(A.packed, A.L, 1, W, nullptr, A.thresh, A.rk, ctr1, nullptr, 4u,
                                                    true, row, lane, tm, tk, tn, sS, sB, 0, s_mask[wq]);
                else if (st)
                    ferro_strip<2, 1, true, false>(A.packed, A.L, 1, W, nullptr, A.thresh, A.rk, ctr1, nullptr, 4u,
                                                   true, row, lane, tm, tk, tn, sS, sB, 0, s_mask[wq]);
                else
                    ferro_strip<2, 1, false, false>(A.packed, A.L, 1, W, nullptr, A.thresh, A.rk, ctr1, nullptr, 4u,
                                                    true, row, lane, tm, tk, tn, sS, sB, 0, s_mask[wq]);
            } else {
                for (int w = lane; w < W; w += 32)
                    resident_word<kMode, kFerro>(A, own, oth, w, color, k, ctr1, sS, sB, st,
                                                 kFerro ? s_mask[wq] : nullptr, wr_shift);
            }
            __syncwarp();  // the colour's words are stored before the other colour reads them
        }
        if (!need_stats) continue;
        sS = __reduce_add_sync(0xffffffffu, sS);
        sB = __reduce_add_sync(0xffffffffu, sB);
        int nk = k;
        if (lane == 0) {
            const int64_t S = sS, Bd = sB;
            const int64_t round = exch ? done / A.swap_every - 1 : 0;
            uint64_t* const slot_word = ring + (round % kRing) * (int64_t)R;
            if (exch) {  // first: the partner is waiting for it
                const uint64_t mine = p2p_pack(S, Bd, round);
                if (multi) {
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
                const int64_t col = done / A.record_every - 1;
                A.obs_e[(int64_t)k * A.ncols + col] = __dsub_rn(__dmul_rn(A.B, (double)S), __dmul_rn(A.J, (double)Bd));
                A.obs_m[(int64_t)k * A.ncols + col] = __ddiv_rn((double)S, (double)A.L * A.L);
            }
            const int first = (int)(round % 2), n_pairs = (R - first) / 2;
            if (exch && k >= first && (k - first) / 2 < n_pairs) {
                {
                    // everything that does not need the partner's energy, while its word travels
                    // (loaded here rather than before the sweep: held across the
                    // strip code, the values cost the 64-register build spills)
                    const int p = (k - first) / 2, i = first + 2 * p, other = k == i ? i + 1 : i;
                    const double u = A.u_table[(round - A.u_round0) * A.u_stride + p];
                    const double bi = A.betas[i], bj = A.betas[i + 1];
                    const uint32_t ot3 = kFerro ? __ldg(A.thresh + other * 10 + 8) : 0u;
                    const uint32_t ot4 = kFerro ? __ldg(A.thresh + other * 10 + 9) : 0u;
                    const uint64_t want = (uint64_t)((round & 0x7fff) | 0x8000);
                    uint64_t v = multi ? ld_relaxed_sys_u64(slot_word + other) : ld_relaxed_u64(slot_word + other);
                    while ((v & 0xffffull) != want) {
                        __nanosleep(64);
                        v = multi ? ld_relaxed_sys_u64(slot_word + other) : ld_relaxed_u64(slot_word + other);
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
                        s_slot[wq] = nk;
                        if (kFerro) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const uint32_t ta = (ot3 >> (31 - q)) & 1u, tb = (ot4 >> (31 - q)) & 1u;
                                s_mask[wq][q] = tb - ta;
                                s_mask[wq][8 + q] = 0u - ta;
                            }
                            s_mask[wq][16] = ot3;
                            s_mask[wq][17] = ot4;
                            s_mask[wq][18] = (uint32_t)nk;
                        }
                    }
                }
            }
        }
        if (exch) ++rounds;
        k = __shfl_sync(0xffffffffu, nk, 0);
        __syncwarp();  // s_mask of the new slot before the next sweep
    }
    // the permutation is an output only: the final mapping, in the buffer the
    // grid-barrier kernel would leave it in (buf flips once per round)
    if (lane == 0) {
        const int fb = A.buf ^ (rounds & 1);
        A.r2s[fb][row] = k;
        A.s2r[fb][k] = A.row_lo + row;
    }
}

template <int kMode, bool kFerro, int kThreads>
static int launch_resident_t(const ResidentArgs& a, int sms, cudaStream_t s) {
    int per_sm = 0;
    PTMH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, cb_resident_kernel<kMode, kFerro, kThreads, false>, kThreads, 0));
    const int slots = a.max_ctas > 0 ? std::min(a.max_ctas, sms * std::max(1, per_sm)) : sms * std::max(1, per_sm);
    // Fewer lattices than CTA slots and enough words per lattice: a cluster
    // of cs CTAs owns each lattice (C2: 64 lattices of 1024 words per colour
    // on 4-CTA clusters of 256 threads, two CTAs per SM).  Measured at C2 with
    // a round every sweep: 1 CTA per lattice 8.80 us/sweep, clusters of 2
    // 7.20, 4 6.93, 8 7.01.  PTMH_RESIDENT_CLUSTER=1 turns it off.
    int cs = 1;
    const char* ec = getenv("PTMH_RESIDENT_CLUSTER");  // "1": off; "2", "4", "8": that size
    if (ec && atoi(ec) > 1) {
        cs = atoi(ec);
    } else if (!(ec && ec[0] == '1') && kThreads == 1024) {
        while (cs < 8 && (int64_t)a.R * cs * 2 <= 2 * slots && a.W / (cs * 2) >= 256) cs *= 2;
    }
    // enough blocks to fill the GPU, few enough that no block owns more
    // lattices than its shared-memory tables hold
    // ONE CTA for every lattice of a tiny run (its rounds then need a CTA
    // barrier instead of a grid barrier) only on request: with the
    // point-to-point rounds, spreading the lattices over the SMs measured
    // faster for every small shape (us per sweep + round, one CTA -> spread:
    // 32^2 x 8 (C1) 2.63 -> 2.40, 64^2 x 16 4.46 -> 2.94, 64^2 x 64 21.0 ->
    // 3.0, 128^2 x 16 21.0 -> 5.1).  PTMH_RESIDENT_ONECTA=1 forces it (A/B).
    for (;; cs = std::max(1, cs / 2)) {
        const char* eo = getenv("PTMH_RESIDENT_ONECTA");
        const bool one_cta = cs == 1 && (int64_t)a.R * a.W <= 4 * kThreads && a.R <= kMaxLatPerBlock &&
                             eo && eo[0] == '1';
        const int grid = cs > 1 ? a.R * cs : (one_cta ? 1 : std::min(a.R, slots));
        if (cs == 1 && (a.R + grid - 1) / grid > kMaxLatPerBlock) {
            set_error("resident kernel: too many lattices per block for this grid");
            return PTMH_ERR_ARG;
        }
        // as few threads as keep the item loop's trip count: every thread then
        // does the same number of words per colour (no tail warps at the barrier)
        const int64_t items = (int64_t)((a.R * cs + grid - 1) / grid) * a.W / cs;
        const int64_t trips = (items + kThreads - 1) / kThreads;
        int threads = (int)std::min<int64_t>(kThreads, (((items + trips - 1) / trips) + 31) & ~31);
        ResidentArgs args = a;
        // warp-owned lattices when a lattice is at most 2 words per lane per
        // colour and the CTA's lattices fit its warps (C5: 28 lattices of 64
        // words per CTA); PTMH_RESIDENT_WARPLAT=0 turns it off (A/B)
        const char* ew = getenv("PTMH_RESIDENT_WARPLAT");
        const int nl_max = (a.R + grid - 1) / grid;
        args.warp_lat = cs == 1 && !(ew && ew[0] == '0') && a.W <= 64 && nl_max <= kThreads / 32;
        if (args.warp_lat) threads = 32 * nl_max;
        // L = 64 (one word per colour row): the lane-per-2-row-strip code of the
        // sweep kernels; PTMH_RESIDENT_STRIP=0 keeps the per-word code (A/B)
        const char* es = getenv("PTMH_RESIDENT_STRIP");
        args.strip = args.warp_lat && a.ferro && a.W == 64 && a.WR == 1 && !(es && es[0] == '0');
        void* kargs[] = {&args};
        if (args.strip) {  // 64^2 ferro lattices: held in registers (resident_reg.cu)
            const int rc = launch_cb_resident_reg64(args, grid, threads, s);
            if (rc != 1) return rc;
        }
        if (args.warp_lat && a.ferro && a.L == 32) {  // 32^2 ferro lattices (C1): the same
            const int rc = launch_cb_resident_reg32(args, grid, threads, s);
            if (rc != 1) return rc;
        }
        // point-to-point rounds (cb_resident_p2p_kernel): warp-owned lattices, one
        // per warp, one GPU, a swap-draw table; PTMH_RESIDENT_P2P=0 turns it off
        const char* ep = getenv("PTMH_RESIDENT_P2P");
        if (cs == 1 && args.warp_lat && a.u_table && nl_max <= threads / 32 && a.L <= 1024 &&
            !(ep && ep[0] == '0')) {
            // one GPU: zero the ring (entries of an earlier launch could carry a
            // matching stamp).  Across GPUs other ranks may already be storing
            // into it: a run's ring starts zeroed (ptmh_peer_alloc) and its round
            // indices only grow, so an older entry never matches
            if (a.swap_every > 0 && a.world == 1)
                PTMH_CUDA(cudaMemsetAsync(a.slot_stats, 0, (size_t)kRing * a.R * 8, s));
            PTMH_CUDA(cudaLaunchCooperativeKernel((const void*)cb_resident_p2p_kernel<kMode, kFerro, kThreads>, grid,
                                                  threads, kargs, 0, s));
            cb_set_last_launch(CbLaunchInfo{6, 1, threads, 1, 0, grid});
            return PTMH_OK;
        }
        if (cs == 1) {
            PTMH_CUDA(cudaLaunchCooperativeKernel((const void*)cb_resident_kernel<kMode, kFerro, kThreads, false>, grid,
                                                  threads, kargs, 0, s));
            cb_set_last_launch(CbLaunchInfo{5, 1, threads, 1, 0, grid});
            return PTMH_OK;
        }
        if (a.u_table && a.world == 1 && a.L <= 1024 && !(ep && ep[0] == '0')) {
            args.p2p = 1;  // cluster-owned lattices: point-to-point rounds
            if (a.swap_every > 0) PTMH_CUDA(cudaMemsetAsync(a.slot_stats, 0, (size_t)kRing * a.R * 8, s));
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3((unsigned)threads);
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeCooperative;
        attr[1].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        // cluster CTAs of <= 256 threads (C2): the 256-thread build (<= 128
        // registers, two CTAs per SM) instead of the 64-register 1024-thread one
        const void* fn = threads <= 256 ? (const void*)cb_resident_kernel<kMode, kFerro, 256, true>
                                        : (const void*)cb_resident_kernel<kMode, kFerro, kThreads, true>;
        const cudaError_t le = cudaLaunchKernelExC(&cfg, fn, kargs);
        if (le == cudaErrorCooperativeLaunchTooLarge) {
            // every cluster must be resident at once; cluster placement can
            // refuse a grid the SM count admits (1024^2 x 32 on 4-CTA clusters
            // of 1024 threads): retry on smaller clusters, finally on CTAs
            cudaGetLastError();
            continue;
        }
        PTMH_CUDA(le);
        cb_set_last_launch(CbLaunchInfo{args.p2p ? 7 : 5, cs, threads, 1, 0, grid});
        return PTMH_OK;
    }
}

template <int kMode, bool kFerro>
static int launch_resident_sized(const ResidentArgs& a, cudaStream_t s) {
    int dev = 0, sms = 0;
    PTMH_CUDA(cudaGetDevice(&dev));
    PTMH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // One 1024-thread CTA per SM: the per-round grid barrier then has the
    // fewest participants (measured on B200: C5 +6%, C3 +12% over 256-thread
    // CTAs).  Fall back to narrower CTAs only when a CTA would own more
    // lattices than its shared tables hold.
    if (const char* e = getenv("PTMH_RESIDENT_THREADS")) {  // tuning override
        if (atoi(e) == 256) return launch_resident_t<kMode, kFerro, 256>(a, sms, s);
    }
    int per_sm = 0;
    PTMH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, cb_resident_kernel<kMode, kFerro, 1024, false>, 1024, 0));
    const int64_t grid = std::min<int64_t>(a.R, (int64_t)sms * std::max(1, per_sm));
    if ((a.R + grid - 1) / grid <= kMaxLatPerBlock) return launch_resident_t<kMode, kFerro, 1024>(a, sms, s);
    return launch_resident_t<kMode, kFerro, 256>(a, sms, s);
}

int64_t resident_ws_bytes(int64_t R, int64_t n_rounds) { return std::max<int64_t>(1, n_rounds) * (R / 2 + 1) * 8; }

int launch_cb_resident(const ResidentArgs& a_in, bool fast, cudaStream_t s, int* grid_out) {
    (void)grid_out;
    ResidentArgs a = a_in;
    if (a.u_table && a.swap_every > 0) {  // this segment's swap draws, for the point-to-point rounds
        // rounds fire at done = (r + 1) * swap_every, first_sweep < done <= the
        // segment's end, strictly below total_sweeps (executor.py:111-125)
        const int64_t last = std::min(a.first_sweep + a.n_sweeps, a.total_sweeps - 1);
        const int64_t n = a.u_stride * std::max<int64_t>(1, last / a.swap_every - a.u_round0);
        swap_draws_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(
            a.seed, a.world > 1 ? a.R_total : a.R, a.u_round0, n / a.u_stride, a.u_stride,
            const_cast<double*>(a.u_table));
        PTMH_LAUNCH_CHECK();
    }
    const bool segs = !fast && a.L >= 8 && 64 % a.L == 0;
    if (segs) {
        const int seg = a.L / 2;
        a.seg_lo = 0;
        a.seg_even = 0;
        for (int b = 0; b < 32; b += seg) {
            a.seg_lo |= 1u << b;
            if (((b / seg) & 1) == 0) a.seg_even |= (seg == 32 ? 0xffffffffu : ((1u << seg) - 1u)) << b;
        }
    }
    if (fast && a.ferro) {  // cluster-owned lattices held in shared memory (resident_smem.cu)
        const int rc = launch_cb_cluster_smem(a, s);
        if (rc != 1) return rc;
    }
    if (fast)
        return a.ferro ? launch_resident_sized<kGatherRows, true>(a, s)
                       : launch_resident_sized<kGatherRows, false>(a, s);
    if (segs)
        return a.ferro ? launch_resident_sized<kGatherSegments, true>(a, s)
                       : launch_resident_sized<kGatherSegments, false>(a, s);
    return a.ferro ? launch_resident_sized<kGatherGeneric, true>(a, s)
                   : launch_resident_sized<kGatherGeneric, false>(a, s);
}

}  // namespace ptmh

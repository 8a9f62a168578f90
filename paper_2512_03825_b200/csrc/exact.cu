// exact.cu -- the reference's random-site chain on the GPU, bit-exact.
//
// Kernels (reference file:line they reproduce):
//   fill_kernel          kernels.py:26-45   exact-count Fisher-Yates init
//   row_stats_kernel     kernels.py:48-59   integer energy / spin-sum accumulators
//   advance_kernel       kernels.py:62-113  random-site MH, incremental E / sum(s)
//                                           (single pass; full_states recording)
//   draw_kernel +        kernels.py:62-113  two phases: every draw / site /
//   commit_kernel                           acceptance bit in parallel, then a
//                                           warp-per-slot commit in 32-windows
//   draw_w_kernel +      kernels.py:62-113  integer J, B, L >= 16: 1024-attempt
//   commit_w_kernel<rec>                    CTA windows (free attempts in one
//                                           pass, dependents in order)
//   exact_resident_kernel executor.py:227-262 + the above: <= 32 slots, every
//                                           lattice in shared memory, swap
//                                           rounds inside the launch
//   swap_kernel          kernels.py:116-148 logistic replica exchange (labels only)
//
// Parallelism.  The reference chain is sequential per slot, but its draws are
// state-independent: attempt a of slot k uses the Philox4x64-10 words at
// positions pos+2a and pos+2a+1 whether or not earlier flips were accepted
// (kernels.py:84-87).  One warp owns a slot and evaluates 32 consecutive
// attempts per window: every lane computes its two draws and its site in
// parallel; attempt a depends on an earlier attempt a' of the window only if
// a' writes a site a reads (same site or a nearest neighbour), so the window
// is committed in dependency levels.  Energies are summed in attempt order
// (exactly, with an order-free integer scan when J and B are integers).
//
// Compiled with -fmad=false: the reference's FP64 expressions are evaluated
// without FMA contraction; every FP op below is also spelled with _rn
// intrinsics where contraction would otherwise be possible.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "launchers.cuh"
#include "philox.cuh"
#include "rounds.cuh"

namespace ptmh {

#define PTMH_TRY_RC(expr)               \
    do {                                \
        int rc_ = (expr);               \
        if (rc_ != PTMH_OK) return rc_; \
    } while (0)

constexpr unsigned kFull = 0xffffffffu;

// ----------------------------------------------------------------- init --
// One warp per lattice row r (stream stream0 + r).  Lanes generate 32 draws
// of the Fisher-Yates sequence in parallel; lane 0 applies the swaps in order.
template <bool kSmem>
__global__ void fill_kernel(int8_t* __restrict__ spins, int64_t rows, int64_t n,
                            int64_t up_count, uint64_t seed, uint64_t stream0,
                            uint64_t pos0) {
    extern __shared__ int8_t smem_lat[];
    __shared__ int64_t jbuf[32];
    const int lane = threadIdx.x & 31;
    const int64_t row = blockIdx.x;
    if (row >= rows) return;
    int8_t* g = spins + row * n;
    int8_t* a = kSmem ? smem_lat : g;
    for (int64_t t = lane; t < n; t += 32) a[t] = (t < up_count) ? 1 : -1;
    __syncwarp();
    const uint64_t stream = stream0 + (uint64_t)row;
    // step s (0-based) handles i = n-1-s, consuming draw pos0 + s
    for (int64_t s0 = 0; s0 < n - 1; s0 += 32) {
        const int64_t s = s0 + lane;
        const int64_t i = n - 1 - s;
        if (s < n - 1) {
            const double u = stream_uniform(seed, stream, pos0 + (uint64_t)s);
            jbuf[lane] = (int64_t)__dmul_rn(u, (double)(i + 1));
        }
        __syncwarp();
        if (lane == 0) {
            const int cnt = (int)min((int64_t)32, n - 1 - s0);
            for (int k = 0; k < cnt; ++k) {
                const int64_t ii = n - 1 - (s0 + k);
                const int64_t jj = jbuf[k];
                const int8_t tmp = a[ii];
                a[ii] = a[jj];
                a[jj] = tmp;
            }
        }
        __syncwarp();
    }
    if (kSmem) {
        for (int64_t t = lane; t < n; t += 32) g[t] = a[t];
    }
}

// -------------------------------------------------------------- row stats --
__global__ void row_stats_kernel(const int8_t* __restrict__ spins, int64_t L,
                                 int64_t* __restrict__ stats) {
    const int64_t row = blockIdx.x;
    const int8_t* s = spins + row * L * L;
    long long bond = 0, total = 0;
    for (int64_t t = threadIdx.x; t < L * L; t += blockDim.x) {
        const int64_t r = t / L, c = t - r * L;
        const int v = s[t];
        bond += v * (s[((r + 1) % L) * L + c] + s[r * L + (c + 1) % L]);
        total += v;
    }
    for (int o = 16; o > 0; o >>= 1) {
        bond += __shfl_down_sync(kFull, bond, o);
        total += __shfl_down_sync(kFull, total, o);
    }
    __shared__ long long sb[32], st[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { sb[w] = bond; st[w] = total; }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long B = 0, T = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { B += sb[k]; T += st[k]; }
        stats[2 * row] = T;
        stats[2 * row + 1] = B;
    }
}

// ---------------------------------------------------------------- advance --


__global__ void advance_kernel(AdvanceArgs A) {
    const int lane = threadIdx.x & 31;
    const int64_t slot = A.lo + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (slot >= A.hi) return;  // whole warp exits together
    const int64_t L = A.L, n_sites = L * L;
    int8_t* lat = A.spins + A.slot_to_row[slot] * n_sites;
    const double* tbl = A.tbl + slot * 10;
    double e = A.energies[slot];
    long long ssum = A.spin_sums[slot];
    const uint64_t pos0 = A.positions[slot];
    const uint64_t st = (uint64_t)slot + A.stream_offset;
    const double nsd = (double)n_sites;

    for (int64_t w0 = 0; w0 < A.nsteps; w0 += 32) {
        const int64_t a = w0 + lane;  // attempt offset within this call
        const bool valid = a < A.nsteps;
        const int nvalid = (int)min((int64_t)32, A.nsteps - w0);
        // --- state-independent part: two draws and the site (kernels.py:83-93)
        const uint64_t p = pos0 + 2 * (uint64_t)a;
        const double u_site = stream_uniform(A.seed, st, p);
        const double u_acc = stream_uniform(A.seed, st, p + 1);
        const int64_t site = (int64_t)__dmul_rn(u_site, nsd);
        const int64_t r = site / L, c = site - r * L;
        const int64_t up = ((r + 1) % L) * L + c;
        const int64_t dn = ((r - 1 + L) % L) * L + c;
        const int64_t rt = r * L + (c + 1) % L;
        const int64_t lf = r * L + (c - 1 + L) % L;
        // --- dependencies on earlier attempts of the window
        unsigned conf = 0;
        if (A.record == 2) {
            conf = (1u << lane) - 1u;  // full serialisation: snapshot per attempt
        } else {
#pragma unroll 4
            for (int k = 0; k < 32; ++k) {
                const int64_t s2 = __shfl_sync(kFull, site, k);
                const bool hit = (s2 == site) | (s2 == up) | (s2 == dn) | (s2 == rt) | (s2 == lf);
                conf |= (hit && k < lane) ? (1u << k) : 0u;
            }
        }
        // --- commit in dependency levels (kernels.py:88-102)
        unsigned pending = __ballot_sync(kFull, valid);
        double my_d = -0.0;  // IEEE identity: keeps a reference -0.0 energy intact
        int my_ds = 0;
        bool my_acc = false;
        while (pending) {
            const bool ready = ((pending >> lane) & 1u) && ((conf & pending) == 0u);
            if (ready) {
                const int s = lat[site];
                const int nb = lat[up] + lat[dn] + lat[rt] + lat[lf];
                const int cls = (s > 0 ? 5 : 0) + (nb + 4) / 2;
                const double d = A.dcls[cls];
                const bool acc = (d <= 0.0) || (u_acc < tbl[cls]);
                if (acc) {
                    lat[site] = (int8_t)(-s);
                    my_d = d;
                    my_ds = -2 * s;
                    my_acc = true;
                }
            }
            __syncwarp();
            const unsigned rdy = __ballot_sync(kFull, ready);
            pending &= ~rdy;
            if (A.record == 2) {
                // exactly one attempt committed; copy the lattice (kernels.py:106-109)
                const int k = __ffs(rdy) - 1;
                int8_t* dst = A.states + ((slot * A.ncols) + A.start_iter + w0 + k) * n_sites;
                for (int64_t t = lane; t < n_sites; t += 32) dst[t] = lat[t];
                __syncwarp();
            }
        }
        // --- energy and spin sum in attempt order
        const unsigned accm = __ballot_sync(kFull, my_acc && valid);
        int ds_scan = my_ds;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(kFull, ds_scan, o);
            if (lane >= o) ds_scan += v;
        }
        const long long ssum_lane = ssum + ds_scan;
        double e_lane;
        if (A.int_energy) {
            // integer-valued increments: any summation order is exact
            double d_scan = my_d;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double v = __shfl_up_sync(kFull, d_scan, o);
                if (lane >= o) d_scan = __dadd_rn(d_scan, v);
            }
            const bool any_before = (accm & ((2u << lane) - 1u)) != 0u;
            e_lane = any_before ? __dadd_rn(e, d_scan) : e;
        } else {
            double run = e;
            e_lane = e;
            for (int k = 0; k < nvalid; ++k) {
                const double dk = __shfl_sync(kFull, my_d, k);
                if ((accm >> k) & 1u) run = __dadd_rn(run, dk);
                if (lane == k) e_lane = run;
            }
        }
        if (A.record >= 1 && valid) {
            const int64_t col = A.start_iter + a;
            A.obs_e[slot * A.ncols + col] = e_lane;
            A.obs_m[slot * A.ncols + col] = __ddiv_rn((double)ssum_lane, nsd);
        }
        e = __shfl_sync(kFull, e_lane, nvalid - 1);
        ssum = __shfl_sync(kFull, ssum_lane, nvalid - 1);
    }
    if (lane == 0) {
        A.energies[slot] = e;
        A.spin_sums[slot] = ssum;
        A.positions[slot] = pos0 + 2 * (uint64_t)A.nsteps;
        A.iters_done[slot] = A.start_iter + A.nsteps;
    }
}

// ---------------------------------------------- two-phase advance (draws) --
// Phase 1: one thread per attempt.  Everything about an attempt that does not
// depend on the lattice state is computed here, fully parallel over slots and
// attempts: the two Philox4x64-10 words (kernels.py:84-87), the site
// (kernels.py:88-90), one acceptance bit per uphill class
// (u_acc < exp(-beta*dE_c), kernels.py:95-98), the mask of earlier attempts of
// the same 32-attempt window whose site is the site or one of its neighbours,
// and per 128-attempt super-window a flag "no two of its sites are within
// Chebyshev distance 1" (then its attempts commute and phase 2 applies them
// in one parallel pass).
// row of site x (0 <= x < L*L <= 2^24 for the two-phase kernels): float
// reciprocal estimate, then an exact +-1 correction
__device__ __forceinline__ int site_row(int x, int L, float invL) {
    int r = (int)__fmul_rn((float)x, invL);
    r -= (r * L > x);
    r += ((r + 1) * L <= x);
    return r;
}

constexpr int kSW = 128;       // attempts per super-window (4 windows)
constexpr int kHashSlots = 512;

struct DrawArgs {
    int64_t lo, nslots, L;
    const double* tbl;
    const double* dcls;
    uint64_t seed;
    const uint64_t* positions;  // call-start positions (by slot)
    int64_t a0, n, stride;      // attempts [a0, a0+n) of the call; record stride
    int32_t* rec_site;
    uint32_t* rec_acc;
    uint32_t* rec_conf;
    uint32_t* rec_indep;        // (nslots, stride / kSW)
};

__global__ void __launch_bounds__(256) draw_kernel(DrawArgs D) {
    __shared__ uint32_t h_tab[2][4][kHashSlots];
    __shared__ int h_dep[2];
    const int64_t npad = (D.n + kSW - 1) / kSW * kSW;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t s = tid / npad;
    const bool in_slot = s < D.nslots;  // no early return: block barriers below
    const int64_t a = in_slot ? tid - s * npad : 0;
    const int lane = threadIdx.x & 31, half = threadIdx.x / kSW;
    for (int k = threadIdx.x; k < 2 * 4 * kHashSlots; k += blockDim.x) (&h_tab[0][0][0])[k] = 0xffffffffu;
    if (threadIdx.x < 2) h_dep[threadIdx.x] = 0;
    __syncthreads();
    const int64_t slot = D.lo + (in_slot ? s : 0);
    const int64_t L = D.L;
    const uint64_t p = D.positions[slot] + 2 * (uint64_t)(D.a0 + a);
    const double u_site = stream_uniform(D.seed, (uint64_t)slot, p);
    const double u_acc = stream_uniform(D.seed, (uint64_t)slot, p + 1);
    const int Li = (int)L;
    const int site = (int)__dmul_rn(u_site, (double)(L * L));
    const int r = site_row(site, Li, 1.0f / (float)Li), c = site - r * Li;
    uint32_t accm = 0;
    const double* tb = D.tbl + slot * 10;
#pragma unroll
    for (int q = 0; q < 10; ++q)
        if (D.dcls[q] > 0.0 && u_acc < tb[q]) accm |= 1u << q;
    // window dependencies: shifted-2x2-bucket filter (two sites at Chebyshev
    // distance <= 1 share one of 4 buckets), exact neighbour test where it fires
    const unsigned lt_mask = (1u << lane) - 1u;
    const bool full = (L & 1) || L <= 8;
    const int rp = (r + 1 == Li) ? 0 : r + 1, cp = (c + 1 == Li) ? 0 : c + 1;
    const int r1 = r >> 1, c1 = c >> 1, r2 = rp >> 1, c2 = cp >> 1;
    const uint32_t keys[4] = {(uint32_t)((r1 << 16) | c1), (uint32_t)((r2 << 16) | c1),
                              (uint32_t)((r1 << 16) | c2), (uint32_t)((r2 << 16) | c2)};
    unsigned cand = 0xffffffffu;
    if (!full)
        cand = __match_any_sync(0xffffffffu, keys[0]) | __match_any_sync(0xffffffffu, keys[1]) |
               __match_any_sync(0xffffffffu, keys[2]) | __match_any_sync(0xffffffffu, keys[3]);
    cand &= lt_mask;
    unsigned conf = 0;
    if (__any_sync(0xffffffffu, cand != 0)) {
        const int up = rp * Li + c, dn = (r == 0 ? Li - 1 : r - 1) * Li + c;
        const int rt = r * Li + cp, lf = r * Li + (c == 0 ? Li - 1 : c - 1);
#pragma unroll 4
        for (int k = 0; k < 32; ++k) {
            const int s2 = __shfl_sync(0xffffffffu, site, k);
            const bool hit = (s2 == site) | (s2 == up) | (s2 == dn) | (s2 == rt) | (s2 == lf);
            conf |= (hit && ((cand >> k) & 1u)) ? (1u << k) : 0u;
        }
    }
    // super-window independence: insert the 4 bucket keys, any repeat => dependent
    const bool valid = in_slot && a < D.n;
    if (full) {
        if (threadIdx.x % kSW == 0) h_dep[half] = 1;
    } else if (valid) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            uint32_t h = (keys[g] * 0x9E3779B1u) >> (32 - 9);
            while (true) {
                const uint32_t old = atomicCAS(&h_tab[half][g][h], 0xffffffffu, keys[g]);
                if (old == 0xffffffffu) break;
                if (old == keys[g]) {
                    h_dep[half] = 1;
                    break;
                }
                h = (h + 1) & (kHashSlots - 1);
            }
        }
    }
    if (valid) {
        const int64_t o = s * D.stride + a;
        D.rec_site[o] = site;
        D.rec_acc[o] = accm;
        D.rec_conf[o] = conf;
    }
    __syncthreads();
    if (in_slot && threadIdx.x % kSW == 0 && a < D.n)
        D.rec_indep[s * (D.stride / kSW) + a / kSW] = h_dep[half] ? 0u : 1u;
}

// Phase 2: warp per slot.  An independent super-window (and integer J, B and
// no recording, so the energy sum is order-free) is applied in one pass, four
// attempts per lane; otherwise its windows of 32 are committed in dependency
// levels with the energies summed in attempt order exactly as advance_kernel.
struct CommitArgs {
    AdvanceArgs A;
    int64_t a0, n, stride;
    const int32_t* rec_site;
    const uint32_t* rec_acc;
    const uint32_t* rec_conf;
    const uint32_t* rec_indep;
    int last;
};

template <bool kBits>
__global__ void __launch_bounds__(128) commit_kernel(CommitArgs C) {
    const AdvanceArgs& A = C.A;
    const int lane = threadIdx.x & 31;
    const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t slot = A.lo + s;
    if (slot >= A.hi) return;
    const int64_t L = A.L, n_sites = L * L;
    const int64_t nwords = (n_sites + 31) >> 5;
    int8_t* lat = kBits ? nullptr : A.spins + A.slot_to_row[slot] * n_sites;
    uint32_t* latw = kBits ? A.bits + A.slot_to_row[slot] * nwords : nullptr;
    auto spin = [&](int64_t x) -> int {  // +1 / -1
        if (kBits) return 2 * (int)((latw[x >> 5] >> (x & 31)) & 1u) - 1;
        return lat[x];
    };
    auto flip = [&](int64_t x, int sp) {
        if (kBits)  // lanes may flip different bits of one word at once
            atomicXor(&latw[x >> 5], 1u << (x & 31));
        else
            lat[x] = (int8_t)(-sp);
    };
    const int Li = (int)L;
    const float invL = 1.0f / (float)Li;
    auto neighbours = [&](int64_t x, int64_t& up, int64_t& dn, int64_t& rt, int64_t& lf) {
        const int xi = (int)x, r = site_row(xi, Li, invL), c = xi - r * Li;
        up = (r + 1 == Li ? 0 : r + 1) * Li + c;
        dn = (r == 0 ? Li - 1 : r - 1) * Li + c;
        rt = r * Li + (c + 1 == Li ? 0 : c + 1);
        lf = r * Li + (c == 0 ? Li - 1 : c - 1);
    };
    double e = A.energies[slot];
    long long ssum = A.spin_sums[slot];
    const double nsd = (double)n_sites;
    const bool unordered = A.int_energy && A.record == 0;  // order-free sums
    double acc_d = -0.0;  // per-lane partial sums (-0.0: the IEEE identity)
    long long acc_ds = 0;
    const int32_t* rs = C.rec_site + s * C.stride;
    const uint32_t* ra = C.rec_acc + s * C.stride;
    const uint32_t* rc = C.rec_conf + s * C.stride;
    const uint32_t* ri = C.rec_indep + s * (C.stride / kSW);
    for (int64_t sw0 = 0; sw0 < C.n; sw0 += kSW) {
        if (unordered && ri[sw0 / kSW]) {
            // the super-window's attempts touch disjoint neighbourhoods: apply all
            int64_t st[4];
            uint32_t am[4];
            bool on[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t a = sw0 + q * 32 + lane;
                on[q] = a < C.n;
                st[q] = on[q] ? rs[a] : 0;
                am[q] = on[q] ? ra[a] : 0u;
            }
            int sp[4], nb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                int64_t up, dn, rt, lf;
                neighbours(st[q], up, dn, rt, lf);
                sp[q] = spin(st[q]);
                nb[q] = spin(up) + spin(dn) + spin(rt) + spin(lf);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int cls = (sp[q] > 0 ? 5 : 0) + (nb[q] + 4) / 2;
                const double d = A.dcls[cls];
                if (on[q] && ((d <= 0.0) || ((am[q] >> cls) & 1u))) {
                    flip(st[q], sp[q]);
                    acc_d = __dadd_rn(acc_d, d);
                    acc_ds += -2 * sp[q];
                }
            }
            __syncwarp();
            continue;
        }
        for (int64_t w0 = sw0; w0 < min(C.n, sw0 + kSW); w0 += 32) {
            const int64_t a = w0 + lane;
            const bool valid = a < C.n;
            const int nvalid = (int)min((int64_t)32, C.n - w0);
            const int64_t site = valid ? rs[a] : 0;
            const uint32_t accm = valid ? ra[a] : 0u;
            const unsigned conf = valid ? rc[a] : 0u;
            int64_t up, dn, rt, lf;
            neighbours(site, up, dn, rt, lf);
            unsigned pending = __ballot_sync(0xffffffffu, valid);
            double my_d = -0.0;
            int my_ds = 0;
            bool my_acc = false;
            while (pending) {
                const bool ready = ((pending >> lane) & 1u) && ((conf & pending) == 0u);
                if (ready) {
                    const int sp = spin(site);
                    const int nbs = spin(up) + spin(dn) + spin(rt) + spin(lf);
                    const int cls = (sp > 0 ? 5 : 0) + (nbs + 4) / 2;
                    const double d = A.dcls[cls];
                    if ((d <= 0.0) || ((accm >> cls) & 1u)) {
                        flip(site, sp);
                        my_d = d;
                        my_ds = -2 * sp;
                        my_acc = true;
                    }
                }
                __syncwarp();
                pending &= ~__ballot_sync(0xffffffffu, ready);
            }
            if (unordered) {
                acc_d = __dadd_rn(acc_d, my_d);
                acc_ds += my_ds;
                continue;
            }
            const unsigned accmask = __ballot_sync(0xffffffffu, my_acc && valid);
            int ds_scan = my_ds;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, ds_scan, o);
                if (lane >= o) ds_scan += v;
            }
            const long long ssum_lane = ssum + ds_scan;
            double e_lane;
            if (A.int_energy) {
                double d_scan = my_d;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double v = __shfl_up_sync(0xffffffffu, d_scan, o);
                    if (lane >= o) d_scan = __dadd_rn(d_scan, v);
                }
                const bool any_before = (accmask & ((2u << lane) - 1u)) != 0u;
                e_lane = any_before ? __dadd_rn(e, d_scan) : e;
            } else {
                double run = e;
                e_lane = e;
                for (int k = 0; k < nvalid; ++k) {
                    const double dk = __shfl_sync(0xffffffffu, my_d, k);
                    if ((accmask >> k) & 1u) run = __dadd_rn(run, dk);
                    if (lane == k) e_lane = run;
                }
            }
            if (A.record >= 1 && valid) {
                const int64_t col = A.start_iter + C.a0 + a;
                A.obs_e[slot * A.ncols + col] = e_lane;
                A.obs_m[slot * A.ncols + col] = __ddiv_rn((double)ssum_lane, nsd);
            }
            e = __shfl_sync(0xffffffffu, e_lane, nvalid - 1);
            ssum = __shfl_sync(0xffffffffu, ssum_lane, nvalid - 1);
        }
    }
    if (unordered) {
        for (int o = 16; o > 0; o >>= 1) {
            acc_d = __dadd_rn(acc_d, __shfl_down_sync(0xffffffffu, acc_d, o));
            acc_ds += __shfl_down_sync(0xffffffffu, acc_ds, o);
        }
        e = __dadd_rn(e, acc_d);  // exact (integer-valued); -0.0 when nothing changed
        ssum += acc_ds;
    }
    if (lane == 0) {
        A.energies[slot] = e;
        A.spin_sums[slot] = ssum;
        if (C.last) {
            A.positions[slot] += 2 * (uint64_t)(C.a0 + C.n);
            A.iters_done[slot] = A.start_iter + C.a0 + C.n;
        }
    }
}

// ------------------------------------------ 1024-attempt windows (L >= 16) --
// For integer J, B and no per-attempt recording (the energy sum is then
// order-free) and lattices large enough that attempts rarely touch, a slot's
// attempts are committed 1024 at a time by a whole CTA:
//   * "free" attempts -- no EARLIER attempt of the window writes a site they
//     read (their site or a neighbour) -- are pairwise independent and go in
//     one parallel pass, 4 per thread;
//   * the few "dependent" ones (~2.6 per window at L = 1024) follow in
//     attempt order, 32 at a time, in dependency levels.
// This is the reference order: a free attempt that touches a dependent one is
// always the earlier of the two (otherwise it would not be free).
// draw_w_kernel marks dependents (bit 31 of the acceptance mask) with a
// shared-memory hash of the window's sites -> earliest attempt.
constexpr int kWin = 1024;
constexpr int kWinHash = 4096;  // load 1/4: short warp-wide probe loops (2048: -18 %)

__device__ __forceinline__ int win_hash(int site) { return (int)(((uint32_t)site * 0x9E3779B1u) >> (32 - 12)); }

// The window path's commit needs no 32-window conflict masks (rec_conf is
// not written).  Per attempt: the two draws, the site (a shift for
// power-of-two L, which equals the reference's int(u * L*L) exactly), the
// uphill-class acceptance bits against the slot's table held in shared
// memory, and the dependent flag.
#ifndef PTMH_DRAW_MINB
#define PTMH_DRAW_MINB 3  // 80 registers, no spills (4: 64 + spills, 2% slower)
#endif
// A 64 Kbit filter in front of the hash: most of the 5 lookups per attempt
// (the site and its neighbours) find no attempt of the window there, and the
// filter answers those without a probe loop -- warp-wide, a probe loop runs as
// long as its longest lane (~10 iterations at load 1/2).
constexpr int kWinFilterWords = 2048;

__device__ __forceinline__ uint32_t win_filter_bit(int site) {
    return ((uint32_t)site * 0x85EBCA6Bu) >> 16;  // 16-bit index
}

__global__ void __launch_bounds__(256, PTMH_DRAW_MINB) draw_w_kernel(DrawArgs D) {
    __shared__ int h_key[kWinHash], h_val[kWinHash];
    __shared__ uint32_t s_filter[kWinFilterWords];
    __shared__ double s_tbl[10];
    __shared__ int s_up[10];
    const int64_t nwin = (D.n + kWin - 1) / kWin;
    const int64_t s = blockIdx.x / nwin;  // grid = nslots * nwin
    const int64_t w0 = (blockIdx.x - s * nwin) * kWin;
    const int64_t slot = D.lo + s;
    for (int k = threadIdx.x; k < kWinHash; k += blockDim.x) {
        h_key[k] = -1;
        h_val[k] = 0x7fffffff;
    }
    for (int k = threadIdx.x; k < kWinFilterWords; k += blockDim.x) s_filter[k] = 0u;
    if (threadIdx.x < 10) {
        s_tbl[threadIdx.x] = D.tbl[slot * 10 + threadIdx.x];
        s_up[threadIdx.x] = D.dcls[threadIdx.x] > 0.0;
    }
    __syncthreads();
    const int Li = (int)D.L;
    const float invL = 1.0f / (float)Li;
    const int lg = __ffs(Li) - 1;
    const bool pow2 = (Li & (Li - 1)) == 0;
    const uint64_t pos0 = D.positions[slot] + 2 * (uint64_t)(D.a0 + w0);
    int site[4];
    uint32_t accm[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int li = q * 256 + threadIdx.x;
        const uint64_t p = pos0 + 2 * (uint64_t)li;
        const uint64_t w_site = philox4x64_word0(D.seed, (uint64_t)slot, p);
        const double u_acc = uniform53(philox4x64_word0(D.seed, (uint64_t)slot, p + 1));
        if (pow2)  // int(u * 2^(2 lg)) with u = (w >> 11) 2^-53: the top 2 lg bits of w
            site[q] = lg == 0 ? 0 : (int)(w_site >> (64 - 2 * lg));
        else
            site[q] = (int)__dmul_rn(uniform53(w_site), (double)((int64_t)Li * Li));
        uint32_t am = 0;
#pragma unroll
        for (int cl = 0; cl < 10; ++cl)
            if (s_up[cl] && u_acc < s_tbl[cl]) am |= 1u << cl;
        accm[q] = am;
        if (w0 + li < D.n) {  // site -> earliest attempt of the window
            const uint32_t fb = win_filter_bit(site[q]);
            atomicOr(&s_filter[fb >> 5], 1u << (fb & 31));
            int h = win_hash(site[q]);
            while (true) {
                const int old = atomicCAS(&h_key[h], -1, site[q]);
                if (old == -1 || old == site[q]) {
                    atomicMin(&h_val[h], li);
                    break;
                }
                h = (h + 1) & (kWinHash - 1);
            }
        }
    }
    __syncthreads();
    auto earliest = [&](int x) -> int {
        const uint32_t fb = win_filter_bit(x);
        if (!((s_filter[fb >> 5] >> (fb & 31)) & 1u)) return 0x7fffffff;  // no attempt at x
        int h = win_hash(x);
        while (true) {
            const int k = h_key[h];
            if (k == x) return h_val[h];
            if (k == -1) return 0x7fffffff;
            h = (h + 1) & (kWinHash - 1);
        }
    };
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int li = q * 256 + threadIdx.x;
        if (w0 + li >= D.n) continue;
        const int x = site[q];
        const int r = pow2 ? x >> lg : site_row(x, Li, invL), c = x - r * Li;
        const int rp = (r + 1 == Li) ? 0 : r + 1, cp = (c + 1 == Li) ? 0 : c + 1;
        const bool dep = (earliest(x) < li) | (earliest(rp * Li + c) < li) |
                         (earliest((r == 0 ? Li - 1 : r - 1) * Li + c) < li) | (earliest(r * Li + cp) < li) |
                         (earliest(r * Li + (c == 0 ? Li - 1 : c - 1)) < li);
        const int64_t o = s * D.stride + w0 + li;
        D.rec_site[o] = site[q];
        D.rec_acc[o] = accm[q] | (dep ? 0x80000000u : 0u);
    }
}

// kRec: per-attempt E and M recorded (record 1).  With integer J and B every
// partial sum is exact, so the window's energies in attempt order are a
// CTA-wide prefix sum of the accepted increments (the -0.0 identity and the
// "no accepted attempt yet" rule keep the reference's signed zeros).
//
// kSmem: the slot's bit lattice is copied into shared memory for the call
// (dynamic, nwords words; L <= 1024 at 128 KB) and back at the end, so the
// spin gathers and flips of every window hit shared memory instead of L2:
// the window commit is a chain of dependent loads and atomics (free pass,
// then the dependent attempts level by level).
template <bool kRec, bool kSmem>
__global__ void __launch_bounds__(256) commit_w_kernel(CommitArgs C) {
    extern __shared__ uint32_t s_latw[];
    __shared__ uint32_t dep_bits[kWin / 32];
    __shared__ double s_d[kRec ? kWin : 1];
    __shared__ int s_ds[kRec ? kWin : 1];
    __shared__ double w_d[8];
    __shared__ long long w_ds[8];
    __shared__ int w_cnt[8];
    __shared__ int dep_list[kWin];
    __shared__ double red_d[8];
    __shared__ long long red_s[8];
    const AdvanceArgs& A = C.A;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t s = blockIdx.x;
    const int64_t slot = A.lo + s;
    const int Li = (int)A.L;
    const float invL = 1.0f / (float)Li;
    const int64_t nwords = ((int64_t)Li * Li + 31) >> 5;
    uint32_t* const latw_g = A.bits + A.slot_to_row[slot] * nwords;
    if (kSmem) {
        for (int64_t k = threadIdx.x; k < nwords; k += blockDim.x) s_latw[k] = latw_g[k];
        // (ordered before the first gather by the window loop's first barrier)
    }
    uint32_t* latw = kSmem ? s_latw : latw_g;
    auto spin = [&](int x) -> int { return 2 * (int)((latw[x >> 5] >> (x & 31)) & 1u) - 1; };
    auto nbrs = [&](int x, int& up, int& dn, int& rt, int& lf) {
        const int r = site_row(x, Li, invL), c = x - r * Li;
        up = (r + 1 == Li ? 0 : r + 1) * Li + c;
        dn = (r == 0 ? Li - 1 : r - 1) * Li + c;
        rt = r * Li + (c + 1 == Li ? 0 : c + 1);
        lf = r * Li + (c == 0 ? Li - 1 : c - 1);
    };
    double acc_d = -0.0;  // IEEE identity (see commit_kernel)
    long long acc_ds = 0;
    double e_run = kRec ? A.energies[slot] : 0.0;  // energy / spin sum before the window
    long long s_run = kRec ? A.spin_sums[slot] : 0;
    const double nsd = (double)((int64_t)Li * Li);
    const int32_t* rs = C.rec_site + s * C.stride;
    const uint32_t* ra = C.rec_acc + s * C.stride;
    // the next window's records are loaded while this one commits
    int nst[4];
    uint32_t nam[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t a = q * 256 + threadIdx.x;
        nst[q] = a < C.n ? rs[a] : 0;
        nam[q] = a < C.n ? ra[a] : 0u;
    }
    for (int64_t w0 = 0; w0 < C.n; w0 += kWin) {
        if (threadIdx.x < kWin / 32) dep_bits[threadIdx.x] = 0;
        if (kRec)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                s_d[q * 256 + threadIdx.x] = -0.0;
                s_ds[q * 256 + threadIdx.x] = 0;
            }
        __syncthreads();
        // ---- free attempts: one parallel pass
        int st[4];
        uint32_t am[4];
        bool on[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t a = w0 + q * 256 + threadIdx.x;
            on[q] = a < C.n;
            st[q] = nst[q];
            am[q] = nam[q];
            const int64_t an = a + kWin;
            nst[q] = an < C.n ? rs[an] : 0;
            nam[q] = an < C.n ? ra[an] : 0u;
        }
        int sp[4], nb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int up, dn, rt, lf;
            nbrs(st[q], up, dn, rt, lf);
            sp[q] = spin(st[q]);
            nb[q] = spin(up) + spin(dn) + spin(rt) + spin(lf);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!on[q]) continue;
            if (am[q] >> 31) {
                const int li = q * 256 + threadIdx.x;
                atomicOr(&dep_bits[li >> 5], 1u << (li & 31));
                continue;
            }
            const int cls = (sp[q] > 0 ? 5 : 0) + (nb[q] + 4) / 2;
            const double d = A.dcls[cls];
            if ((d <= 0.0) || ((am[q] >> cls) & 1u)) {
                atomicXor(&latw[st[q] >> 5], 1u << (st[q] & 31));
                if (kRec) {
                    s_d[q * 256 + threadIdx.x] = d;
                    s_ds[q * 256 + threadIdx.x] = -2 * sp[q];
                } else {
                    acc_d = __dadd_rn(acc_d, d);
                    acc_ds += -2 * sp[q];
                }
            }
        }
        __syncthreads();
        // ---- dependents: warp 0, attempt order, 32 at a time in levels
        if (warp == 0) {
            const uint32_t m = dep_bits[lane];
            int pre = __popc(m);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(kFull, pre, o);
                if (lane >= o) pre += v;
            }
            const int total = __shfl_sync(kFull, pre, 31);
            int pos = pre - __popc(m);
            for (uint32_t mm = m; mm; mm &= mm - 1) dep_list[pos++] = lane * 32 + __ffs(mm) - 1;
            __syncwarp();
            for (int b0 = 0; b0 < total; b0 += 32) {
                const bool valid = b0 + lane < total;
                const int64_t a = w0 + (valid ? dep_list[b0 + lane] : 0);
                const int x = valid ? rs[a] : -1;
                const uint32_t amk = valid ? ra[a] : 0u;
                int up = 0, dn = 0, rt = 0, lf = 0;
                if (valid) nbrs(x, up, dn, rt, lf);
                unsigned conf = 0;
                for (int k = 0; k < 32; ++k) {
                    const int s2 = __shfl_sync(kFull, x, k);
                    const bool hit = (s2 == x) | (s2 == up) | (s2 == dn) | (s2 == rt) | (s2 == lf);
                    conf |= (hit && k < lane && s2 >= 0) ? (1u << k) : 0u;
                }
                unsigned pending = __ballot_sync(kFull, valid);
                while (pending) {
                    const bool ready = ((pending >> lane) & 1u) && ((conf & pending) == 0u);
                    if (ready) {
                        const int spx = spin(x);
                        const int nbx = spin(up) + spin(dn) + spin(rt) + spin(lf);
                        const int cls = (spx > 0 ? 5 : 0) + (nbx + 4) / 2;
                        const double d = A.dcls[cls];
                        if ((d <= 0.0) || ((amk >> cls) & 1u)) {
                            atomicXor(&latw[x >> 5], 1u << (x & 31));
                            if (kRec) {
                                s_d[a - w0] = d;
                                s_ds[a - w0] = -2 * spx;
                            } else {
                                acc_d = __dadd_rn(acc_d, d);
                                acc_ds += -2 * spx;
                            }
                        }
                    }
                    __syncwarp();
                    pending &= ~__ballot_sync(kFull, ready);
                }
            }
        }
        __syncthreads();
        if (kRec) {
            // prefix over the window in attempt order: thread t owns attempts
            // 4t .. 4t+3 (local scan), warps scan thread totals, warp totals
            // are scanned through shared memory
            double ld[4];
            int lds[4], lcnt[4];
            double run_d = -0.0;
            int run_ds = 0, run_c = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = 4 * (int)threadIdx.x + j;
                run_d = __dadd_rn(run_d, s_d[k]);
                run_ds += s_ds[k];
                run_c += s_ds[k] != 0;
                ld[j] = run_d;
                lds[j] = run_ds;
                lcnt[j] = run_c;
            }
            double xd = run_d;  // inclusive scan of thread totals within the warp
            int xds = run_ds, xc = run_c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double vd = __shfl_up_sync(kFull, xd, o);
                const int vds = __shfl_up_sync(kFull, xds, o), vc = __shfl_up_sync(kFull, xc, o);
                if (lane >= o) {
                    xd = __dadd_rn(xd, vd);
                    xds += vds;
                    xc += vc;
                }
            }
            if (lane == 31) {
                w_d[warp] = xd;
                w_ds[warp] = xds;
                w_cnt[warp] = xc;
            }
            __syncthreads();
            double pd = -0.0;  // exclusive prefix of this thread
            long long pds = 0;
            int pc = 0;
            for (int k = 0; k < warp; ++k) {
                pd = __dadd_rn(pd, w_d[k]);
                pds += w_ds[k];
                pc += w_cnt[k];
            }
            {  // exclusive within the warp: the previous lane's inclusive value
                const double ud = __shfl_up_sync(kFull, xd, 1);
                const int uds = __shfl_up_sync(kFull, xds, 1), uc = __shfl_up_sync(kFull, xc, 1);
                if (lane > 0) {
                    pd = __dadd_rn(pd, ud);
                    pds += uds;
                    pc += uc;
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t aa = w0 + 4 * (int)threadIdx.x + j;
                if (aa >= C.n) break;
                const int cnt = pc + lcnt[j];
                const double e_a = cnt > 0 ? __dadd_rn(e_run, __dadd_rn(pd, ld[j])) : e_run;
                const long long s_a = s_run + pds + lds[j];
                const int64_t col = A.start_iter + C.a0 + aa;
                A.obs_e[slot * A.ncols + col] = e_a;
                A.obs_m[slot * A.ncols + col] = __ddiv_rn((double)s_a, nsd);
            }
            double td = -0.0;  // window totals (every thread alike)
            long long tds = 0;
            int tc = 0;
            for (int k = 0; k < 8; ++k) {
                td = __dadd_rn(td, w_d[k]);
                tds += w_ds[k];
                tc += w_cnt[k];
            }
            if (tc > 0) e_run = __dadd_rn(e_run, td);
            s_run += tds;
            __syncthreads();  // w_* and s_d are rewritten by the next window
        }
    }
    // order-free sums (integer-valued d): warp shuffles, then the CTA
    for (int o = 16; o > 0; o >>= 1) {
        acc_d = __dadd_rn(acc_d, __shfl_down_sync(kFull, acc_d, o));
        acc_ds += __shfl_down_sync(kFull, acc_ds, o);
    }
    if (lane == 0) {
        red_d[warp] = acc_d;
        red_s[warp] = acc_ds;
    }
    __syncthreads();
    if (kSmem)  // the window loop's last barrier ordered every flip before this
        for (int64_t k = threadIdx.x; k < nwords; k += blockDim.x) latw_g[k] = s_latw[k];
    if (threadIdx.x == 0) {
        double td = -0.0;
        long long ts = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            td = __dadd_rn(td, red_d[k]);
            ts += red_s[k];
        }
        A.energies[slot] = kRec ? e_run : __dadd_rn(A.energies[slot], td);
        A.spin_sums[slot] = kRec ? s_run : A.spin_sums[slot] + ts;
        if (C.last) {
            A.positions[slot] += 2 * (uint64_t)(C.a0 + C.n);
            A.iters_done[slot] = A.start_iter + C.a0 + C.n;
        }
    }
}

// ----------------------------------------- resident exact run, few slots --
// The reference's C1 shape (8 slots of 32^2, a round every sweep) is bound by
// per-interval launches and by the commit's L2 round trips, not by work.  For
// up to 32 slots whose bit lattices fit in shared memory, ONE CTA commits a
// whole chunk of precomputed draws (draw_kernel records) for every slot --
// warp w = slot w, lattices in shared memory -- and runs the swap rounds that
// fall inside the chunk itself (reference rule, kernels.py:116-148), so a
// chunk of ~64 intervals is one launch.  Windows of 32 attempts are committed
// in dependency levels with energies summed in attempt order, exactly as
// commit_kernel; a round boundary may cut a window (its two parts are
// committed on either side of the round).

template <int kMaxThreads>
__global__ void __launch_bounds__(kMaxThreads, 1) exact_resident_kernel(CommitArgs C, ExactRounds X) {
    extern __shared__ uint32_t s_lat[];  // every lattice, by row, ceil(L*L/32) words each
    __shared__ int s_s2r[32];
    __shared__ double s_e[32];
    __shared__ long long s_ss[32];
    const AdvanceArgs& A = C.A;
    const int R = (int)A.hi;  // lo == 0: every slot
    const int lane = threadIdx.x & 31, slot = threadIdx.x >> 5;
    const int Li = (int)A.L;
    const float invL = 1.0f / (float)Li;
    const int nwords = (Li * Li + 31) >> 5;
    for (int k = threadIdx.x; k < R * nwords; k += blockDim.x) s_lat[k] = A.bits[k];
    if ((int)threadIdx.x < R) {
        s_s2r[threadIdx.x] = (int)A.slot_to_row[threadIdx.x];
        s_e[threadIdx.x] = A.energies[threadIdx.x];
        s_ss[threadIdx.x] = A.spin_sums[threadIdx.x];
    }
    __syncthreads();
    const int64_t it0 = A.start_iter + C.a0;  // iteration of chunk attempt 0
    const int64_t I = X.swap_every;
    const double nsd = (double)(Li * Li);
    const int32_t* rs = C.rec_site + (int64_t)slot * C.stride;
    const uint32_t* ra = C.rec_acc + (int64_t)slot * C.stride;
    const uint32_t* rc = C.rec_conf + (int64_t)slot * C.stride;
    uint32_t* latw = s_lat + (int64_t)s_s2r[slot < R ? slot : 0] * nwords;
    double e = slot < R ? s_e[slot] : 0.0;
    long long ssum = slot < R ? s_ss[slot] : 0;
    // next round: after chunk attempt bnd - 1 (completed = it0 + bnd), if any
    auto next_boundary = [&](int64_t from, int64_t& round) -> int64_t {
        round = -1;
        if (I <= 0) return INT64_MAX;
        const int64_t nb = ((it0 + from) / I + 1) * I;
        if (nb < X.total_iters) round = nb / I - 1;
        return round >= 0 ? nb - it0 : INT64_MAX;
    };
    int64_t round = -1;
    int64_t bnd = next_boundary(0, round);
    // integer J, B and no recording: energies are order-free -- per-lane
    // partial sums, reduced only when a round (or the end) needs them
    const bool unordered = A.int_energy && A.record == 0;
    double acc_d = -0.0;  // IEEE identity (see commit_kernel)
    long long acc_ds = 0;
    auto settle = [&]() {
        if (!unordered) return;
        for (int o = 16; o > 0; o >>= 1) {
            acc_d = __dadd_rn(acc_d, __shfl_xor_sync(kFull, acc_d, o));
            acc_ds += __shfl_xor_sync(kFull, acc_ds, o);
        }
        e = __dadd_rn(e, acc_d);
        ssum += acc_ds;
        acc_d = -0.0;
        acc_ds = 0;
    };
    auto commit = [&](int64_t w0, int64_t lo, int64_t hi, int site, uint32_t accm, unsigned conf) {
        // attempts [lo, hi) of the window at w0 (32-window dependency levels,
        // energies in attempt order: commit_kernel's ordered path)
        const int64_t a = w0 + lane;
        const bool valid = slot < R && a >= lo && a < hi;
        const int last = (int)(hi - w0) - 1;
        auto spin = [&](int x) -> int { return 2 * (int)((latw[x >> 5] >> (x & 31)) & 1u) - 1; };
        const int r = site_row(site, Li, invL), c = site - r * Li;
        const int up = (r + 1 == Li ? 0 : r + 1) * Li + c, dn = (r == 0 ? Li - 1 : r - 1) * Li + c;
        const int rt = r * Li + (c + 1 == Li ? 0 : c + 1), lf = r * Li + (c == 0 ? Li - 1 : c - 1);
        unsigned pending = __ballot_sync(kFull, valid);
        double my_d = -0.0;
        int my_ds = 0;
        bool my_acc = false;
        while (pending) {
            const bool ready = ((pending >> lane) & 1u) && ((conf & pending) == 0u);
            if (ready) {
                const int sp = spin(site);
                const int nbs = spin(up) + spin(dn) + spin(rt) + spin(lf);
                const int cls = (sp > 0 ? 5 : 0) + (nbs + 4) / 2;
                const double d = A.dcls[cls];
                if ((d <= 0.0) || ((accm >> cls) & 1u)) {
                    atomicXor(&latw[site >> 5], 1u << (site & 31));
                    my_d = d;
                    my_ds = -2 * sp;
                    my_acc = true;
                }
            }
            __syncwarp();
            pending &= ~__ballot_sync(kFull, ready);
        }
        if (unordered) {
            if (my_acc) {
                acc_d = __dadd_rn(acc_d, my_d);
                acc_ds += my_ds;
            }
            return;
        }
        const unsigned accmask = __ballot_sync(kFull, my_acc && valid);
        int ds_scan = my_ds;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(kFull, ds_scan, o);
            if (lane >= o) ds_scan += v;
        }
        const long long ssum_lane = ssum + ds_scan;
        double e_lane;
        if (A.int_energy) {
            double d_scan = my_d;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double v = __shfl_up_sync(kFull, d_scan, o);
                if (lane >= o) d_scan = __dadd_rn(d_scan, v);
            }
            const bool any_before = (accmask & ((2u << lane) - 1u)) != 0u;
            e_lane = any_before ? __dadd_rn(e, d_scan) : e;
        } else {
            double run = e;
            e_lane = e;
            for (int k = 0; k <= last; ++k) {
                const double dk = __shfl_sync(kFull, my_d, k);
                if ((accmask >> k) & 1u) run = __dadd_rn(run, dk);
                if (lane == k) e_lane = run;
            }
        }
        if (A.record >= 1 && valid) {
            const int64_t col = it0 + a;
            A.obs_e[(int64_t)slot * A.ncols + col] = e_lane;
            A.obs_m[(int64_t)slot * A.ncols + col] = __ddiv_rn((double)ssum_lane, nsd);
        }
        e = __shfl_sync(kFull, e_lane, last);
        ssum = __shfl_sync(kFull, ssum_lane, last);
    };
    auto do_round = [&](int64_t rnd) {
        settle();
        if (slot < R && lane == 0) {
            s_e[slot] = e;
            s_ss[slot] = ssum;
        }
        __syncthreads();
        if (slot == 0) {  // disjoint pairs, one lane each (kernels.py:116-148)
            const int first = (int)(rnd % 2), n_pairs = (R - first) / 2;
            int acc = 0, ties = 0;
            for (int p = lane; p < n_pairs; p += 32) {
                const int i = first + 2 * p, j = i + 1;
                const double u = stream_uniform(A.seed, (uint64_t)(R + p), (uint64_t)rnd);
                bool near = false;  // (rounds.cuh: FP32 fast path, exact FP64 near the decision)
                const bool accept = swap_decide(__dsub_rn(X.betas[i], X.betas[j]), s_e[i], s_e[j], u, near);
                if (near) ++ties;
                if (accept) {
                    const int tr = s_s2r[i]; s_s2r[i] = s_s2r[j]; s_s2r[j] = tr;
                    const double te = s_e[i]; s_e[i] = s_e[j]; s_e[j] = te;
                    const long long ts = s_ss[i]; s_ss[i] = s_ss[j]; s_ss[j] = ts;
                    ++acc;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                acc += __shfl_down_sync(kFull, acc, o);
                ties += __shfl_down_sync(kFull, ties, o);
            }
            if (lane == 0 && X.counters) {
                if (acc) atomicAdd((unsigned long long*)&X.counters[0], (unsigned long long)acc);
                if (ties) atomicAdd((unsigned long long*)&X.counters[1], (unsigned long long)ties);
            }
        }
        __syncthreads();
        if (slot < R) {
            latw = s_lat + (int64_t)s_s2r[slot] * nwords;
            e = s_e[slot];
            ssum = s_ss[slot];
        }
    };
    // A call covers the rounds at completed = start_iter .. start_iter +
    // nsteps - 1 (each boundary once across consecutive calls): the one at
    // the call's first iteration runs before its first attempt (swap_every =
    // 1: the round after the init iteration), the one at its end belongs to
    // the next call.  Chunk ends inside the call run their boundary's round.
    if (C.a0 == 0 && I > 0 && it0 % I == 0 && it0 >= I && it0 < X.total_iters) do_round(it0 / I - 1);
    // Records stream through registers one group of kGroup windows ahead, so
    // their L2 latency hides behind the current group's commits.
    constexpr int kGroup = 4;
    const int64_t nwin = (C.n + 31) / 32;
    int cs[kGroup], ns[kGroup];
    uint32_t ca[kGroup], na[kGroup], cc[kGroup], nc[kGroup];
#pragma unroll
    for (int q = 0; q < kGroup; ++q) {
        const int64_t a = (int64_t)q * 32 + lane;
        const bool ok = slot < R && a < C.n;
        cs[q] = ok ? rs[a] : 0;
        ca[q] = ok ? ra[a] : 0u;
        cc[q] = ok ? rc[a] : 0u;
    }
    for (int64_t g = 0; g < nwin; g += kGroup) {
#pragma unroll
        for (int q = 0; q < kGroup; ++q) {  // prefetch the next group
            const int64_t a = (g + kGroup + q) * 32 + lane;
            const bool ok = slot < R && a < C.n;
            ns[q] = ok ? rs[a] : 0;
            na[q] = ok ? ra[a] : 0u;
            nc[q] = ok ? rc[a] : 0u;
        }
#pragma unroll
        for (int q = 0; q < kGroup; ++q) {
            const int64_t w0 = (g + q) * 32;
            if (w0 >= C.n) break;
            const int64_t wend = min(w0 + 32, C.n);
            int64_t lo = w0;
            while (lo < wend) {  // rounds may cut the window (several, when I < 32)
                const int64_t hi = min(wend, bnd);
                if (hi > lo) commit(w0, lo, hi, cs[q], ca[q], cc[q]);
                lo = hi;
                if (bnd == hi && hi <= wend) {
                    if (!(C.last && hi == C.n)) do_round(round);
                    bnd = next_boundary(hi, round);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kGroup; ++q) {
            cs[q] = ns[q];
            ca[q] = na[q];
            cc[q] = nc[q];
        }
    }
    settle();
    if (slot < R && lane == 0) {
        s_e[slot] = e;
        s_ss[slot] = ssum;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < R * nwords; k += blockDim.x) A.bits[k] = s_lat[k];
    if ((int)threadIdx.x < R) {
        const_cast<int64_t*>(A.slot_to_row)[threadIdx.x] = s_s2r[threadIdx.x];
        A.energies[threadIdx.x] = s_e[threadIdx.x];
        A.spin_sums[threadIdx.x] = s_ss[threadIdx.x];
        if (C.last) {
            A.positions[threadIdx.x] += 2 * (uint64_t)(C.a0 + C.n);
            A.iters_done[threadIdx.x] = A.start_iter + C.a0 + C.n;
        }
    }
}

int64_t advance_chunk(int64_t nslots) {
    // attempts per slot per phase-1/phase-2 pass: ~16M records (~200 MiB)
    int64_t c = (int64_t(1) << 24) / std::max<int64_t>(1, nslots);
    c = std::max<int64_t>(1024, std::min<int64_t>(c, 1 << 16));
    return c & ~int64_t(kSW - 1);
}

static int64_t advance_stride(int64_t nslots, int64_t nsteps) {
    return std::min(advance_chunk(nslots), (nsteps + kSW - 1) / kSW * kSW);
}

// Two record buffers: the draws of chunk k+1 (issue-bound, fills the GPU) run
// on a side stream while chunk k commits (latency-bound, one warp per slot).
int64_t advance_ws_bytes(int64_t nslots, int64_t nsteps) {
    const int64_t stride = advance_stride(nslots, nsteps);
    const int64_t one = nslots * stride * 12 + nslots * (stride / kSW) * 4;
    return (nsteps > stride ? 2 : 1) * one;
}

// side stream + events for the draw/commit overlap, one set per device
struct DrawStream {
    std::mutex mu;  // held while a call enqueues (the events are shared)
    cudaStream_t s = nullptr;   // draws (default priority)
    cudaStream_t sc = nullptr;  // commits, highest priority: their few CTAs are
                                // placed as soon as draw CTAs retire
    cudaEvent_t drawn[2], committed[2], start;
};

static int draw_stream(DrawStream** out) {
    static std::mutex mu;
    static DrawStream per_dev[64];
    int dev = 0;
    PTMH_CUDA(cudaGetDevice(&dev));
    if (dev >= 64) {
        set_error("advance: device index >= 64");
        return PTMH_ERR_ARG;
    }
    std::lock_guard<std::mutex> lk(mu);
    DrawStream& d = per_dev[dev];
    if (!d.s) {
        PTMH_CUDA(cudaStreamCreateWithFlags(&d.s, cudaStreamNonBlocking));
        int lo_pri = 0, hi_pri = 0;
        PTMH_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
        PTMH_CUDA(cudaStreamCreateWithPriority(&d.sc, cudaStreamNonBlocking, hi_pri));
        for (int b = 0; b < 2; ++b) {
            PTMH_CUDA(cudaEventCreateWithFlags(&d.drawn[b], cudaEventDisableTiming));
            PTMH_CUDA(cudaEventCreateWithFlags(&d.committed[b], cudaEventDisableTiming));
        }
        PTMH_CUDA(cudaEventCreateWithFlags(&d.start, cudaEventDisableTiming));
    }
    *out = &d;
    return PTMH_OK;
}

int launch_advance_2phase(const AdvanceArgs& a, void* ws, int64_t ws_bytes, cudaStream_t s,
                          const ExactRounds* rounds) {
    const int64_t nslots = a.hi - a.lo;
    if (nslots <= 0 || a.nsteps <= 0) return PTMH_OK;
    const int64_t stride = advance_stride(nslots, a.nsteps);
    if (ws_bytes < advance_ws_bytes(nslots, a.nsteps)) {
        set_error("advance workspace too small");
        return PTMH_ERR_ARG;
    }
    const int nbuf = a.nsteps > stride ? 2 : 1;
    // 1024-attempt CTA windows: bit lattices, order-free energy sums, L >= 16
    // (measured against the warp-per-slot commit: 256^2 x 64 slots 2.0e9 ->
    // 1.2e10, 128^2 x 256 4.8e9 -> 1.4e10, 32^2 x 256 3.6e9 -> 4.7e9; equal at 8^2)
    // (PTMH_EXACT_WINDOWS=0 forces the warp path, =2 the window path at any
    // L: A/B in tools/, dependent-heavy windows in tests)
    const char* ew = getenv("PTMH_EXACT_WINDOWS");
    const bool windows = !rounds && a.bits && a.int_energy && a.record <= 1 && a.L <= 4096 &&
                         (ew && ew[0] == '2' ? a.L >= 3 : a.L >= 16) && !(ew && ew[0] == '0');
    // the window commit with the slot's bit lattice in shared memory where it
    // fits (L <= 1024: 128 KB; PTMH_EXACT_LAT_SMEM=0 keeps it in L2, A/B)
    const char* els = getenv("PTMH_EXACT_LAT_SMEM");
    const size_t lat_bytes = (size_t)((a.L * a.L + 31) / 32) * 4;
    const bool lat_smem = windows && lat_bytes <= 160 * 1024 && !(els && els[0] == '0');
    if (lat_smem && lat_bytes > 48 * 1024) {
        PTMH_CUDA(cudaFuncSetAttribute((const void*)commit_w_kernel<true, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lat_bytes));
        PTMH_CUDA(cudaFuncSetAttribute((const void*)commit_w_kernel<false, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lat_bytes));
    }
    size_t res_smem = 0;
    if (rounds) {  // exact_resident_kernel: one CTA, a warp per slot, every lattice in shared memory
        res_smem = (size_t)nslots * (size_t)((a.L * a.L + 31) / 32) * 4;
        if (a.lo != 0 || nslots > 32 || !a.bits || res_smem > 200 * 1024) {
            set_error("resident exact run: needs every slot (<= 32) and bit lattices in shared memory");
            return PTMH_ERR_ARG;
        }
        // instantiations by slot count: <= 8 slots run uncapped (146
        // registers; the 1024-thread one spills at 64: C1 2.2e8 -> 3.9e8)
        const void* fn = nslots <= 8 ? (const void*)exact_resident_kernel<256>
                         : nslots <= 16 ? (const void*)exact_resident_kernel<512>
                                        : (const void*)exact_resident_kernel<1024>;
        PTMH_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
    }
    const int64_t one = nslots * stride * 12 + nslots * (stride / kSW) * 4;
    DrawStream* ds = nullptr;
    std::unique_lock<std::mutex> lk;
    if (nbuf == 2) {
        PTMH_TRY_RC(draw_stream(&ds));
        lk = std::unique_lock<std::mutex>(ds->mu);
        PTMH_CUDA(cudaEventRecord(ds->start, s));  // the draws read positions / tables written on s
        PTMH_CUDA(cudaStreamWaitEvent(ds->s, ds->start, 0));
        PTMH_CUDA(cudaStreamWaitEvent(ds->sc, ds->start, 0));
    }
    cudaStream_t sc = nbuf == 2 ? ds->sc : s;
    int k = 0;
    for (int64_t a0 = 0; a0 < a.nsteps; a0 += stride, ++k) {
        const int b = k % nbuf;
        int32_t* rs = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + b * one);
        uint32_t* ra = reinterpret_cast<uint32_t*>(rs + nslots * stride);
        uint32_t* rc = ra + nslots * stride;
        uint32_t* rind = rc + nslots * stride;
        const int64_t n = std::min(stride, a.nsteps - a0);
        DrawArgs D{a.lo, nslots, a.L, a.tbl, a.dcls, a.seed, a.positions, a0, n, stride, rs, ra, rc, rind};
        const int64_t npad = (n + kSW - 1) / kSW * kSW;
        cudaStream_t sd = nbuf == 2 ? ds->s : s;
        if (nbuf == 2 && k >= 2) PTMH_CUDA(cudaStreamWaitEvent(sd, ds->committed[b], 0));  // buffer free
        const int64_t nwin = (n + kWin - 1) / kWin;
        if (windows)
            draw_w_kernel<<<(unsigned)(nslots * nwin), 256, 0, sd>>>(D);
        else
            draw_kernel<<<ceil_div(nslots * npad, 256), 256, 0, sd>>>(D);
        PTMH_LAUNCH_CHECK();
        if (nbuf == 2) {
            PTMH_CUDA(cudaEventRecord(ds->drawn[b], sd));
            PTMH_CUDA(cudaStreamWaitEvent(sc, ds->drawn[b], 0));
        }
        CommitArgs C{a, a0, n, stride, rs, ra, rc, rind, a0 + n >= a.nsteps};
        if (rounds && nslots <= 8)
            exact_resident_kernel<256><<<1, (unsigned)(32 * nslots), res_smem, sc>>>(C, *rounds);
        else if (rounds && nslots <= 16)
            exact_resident_kernel<512><<<1, (unsigned)(32 * nslots), res_smem, sc>>>(C, *rounds);
        else if (rounds)
            exact_resident_kernel<1024><<<1, (unsigned)(32 * nslots), res_smem, sc>>>(C, *rounds);
        else if (windows && lat_smem && a.record == 1)
            commit_w_kernel<true, true><<<(unsigned)nslots, 256, lat_bytes, sc>>>(C);
        else if (windows && lat_smem)
            commit_w_kernel<false, true><<<(unsigned)nslots, 256, lat_bytes, sc>>>(C);
        else if (windows && a.record == 1)
            commit_w_kernel<true, false><<<(unsigned)nslots, 256, 0, sc>>>(C);
        else if (windows)
            commit_w_kernel<false, false><<<(unsigned)nslots, 256, 0, sc>>>(C);
        else if (a.bits)
            commit_kernel<true><<<ceil_div(nslots, 4), 128, 0, sc>>>(C);
        else
            commit_kernel<false><<<ceil_div(nslots, 4), 128, 0, sc>>>(C);
        PTMH_LAUNCH_CHECK();
        if (nbuf == 2) PTMH_CUDA(cudaEventRecord(ds->committed[b], sc));
    }
    if (nbuf == 2) PTMH_CUDA(cudaStreamWaitEvent(s, ds->committed[(k - 1) % 2], 0));  // join
    return PTMH_OK;
}

// ----------------------------------------------- bit-packed exact lattices --
// Row-major bits (site x -> bit x & 31 of word x >> 5): 1 bit per spin keeps
// the C3 lattices (256 x 1 MiB int8) L2-resident (32 MiB) for the commit.
__global__ void bits_pack_kernel(const int8_t* __restrict__ spins, int64_t rows, int64_t n, int64_t nw,
                                 uint32_t* __restrict__ bits) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * nw) return;
    const int64_t row = t / nw, w = t - row * nw;
    const int8_t* s = spins + row * n;
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b) {
        const int64_t x = w * 32 + b;
        if (x < n && s[x] > 0) word |= 1u << b;
    }
    bits[t] = word;
}

__global__ void bits_unpack_kernel(const uint32_t* __restrict__ bits, int64_t rows, int64_t n, int64_t nw,
                                   int8_t* __restrict__ spins) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * n) return;
    const int64_t row = t / n, x = t - row * n;
    spins[t] = ((bits[row * nw + (x >> 5)] >> (x & 31)) & 1u) ? 1 : -1;
}

int launch_bits_pack(const int8_t* spins, int64_t rows, int64_t L, uint32_t* bits, cudaStream_t s) {
    const int64_t n = L * L, nw = (n + 31) >> 5;
    if (rows == 0) return PTMH_OK;
    bits_pack_kernel<<<ceil_div(rows * nw, 256), 256, 0, s>>>(spins, rows, n, nw, bits);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_bits_unpack(const uint32_t* bits, int64_t rows, int64_t L, int8_t* spins, cudaStream_t s) {
    const int64_t n = L * L, nw = (n + 31) >> 5;
    if (rows == 0) return PTMH_OK;
    bits_unpack_kernel<<<ceil_div(rows * n, 256), 256, 0, s>>>(bits, rows, n, nw, spins);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

// ------------------------------------------------------------------- swap --
// The swap rule's saturating logistic (kernels.py:127-135, tempering.py:53-65)
// in the reference's split form, every operation rounded as numba does.
__device__ __forceinline__ double swap_logistic(double x) {
    if (x >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));
    const double ex = exp(x);
    return __ddiv_rn(ex, __dadd_rn(1.0, ex));
}

// device exp and host libm may differ in the last ulp: a decision such a
// difference could flip is counted (expected: none; every parity test asserts 0)
__device__ __forceinline__ bool near_tie(double u, double prob) {
    return fabs(u - prob) <= 4.0 * 2.220446049250313e-16 * fmax(prob, 2.2250738585072014e-308);
}

__global__ void swap_kernel(int64_t* __restrict__ slot_to_row, double* __restrict__ energies,
                            int64_t* __restrict__ spin_sums, const double* __restrict__ betas,
                            int64_t R, uint64_t seed, int64_t stream_base, int64_t round_index,
                            int64_t first, int64_t pair_lo, int64_t pair_hi,
                            int64_t* accepted, int64_t* near_ties, int32_t* row_to_slot,
                            const int64_t* __restrict__ stats, double J, double B) {
    if (stats) {  // checkerboard chain: by-slot energies from per-lattice (S, Bond) first
        for (int64_t k = threadIdx.x; k < R; k += blockDim.x) {
            const int64_t row = slot_to_row[k];
            const int64_t S = stats[2 * row], Bd = stats[2 * row + 1];
            energies[k] = __dsub_rn(__dmul_rn(B, (double)S), __dmul_rn(J, (double)Bd));
            spin_sums[k] = S;
        }
        __syncthreads();
    }
    int acc = 0, ties = 0;
    for (int64_t p = pair_lo + threadIdx.x; p < pair_hi; p += blockDim.x) {
        const int64_t i = first + 2 * p, j = i + 1;
        const double u = stream_uniform(seed, (uint64_t)(stream_base + p), (uint64_t)round_index);
        const double x = __dmul_rn(__dsub_rn(betas[i], betas[j]), __dsub_rn(energies[i], energies[j]));
        const double prob = swap_logistic(x);
        if (near_tie(u, prob)) ++ties;
        if (u < prob) {
            const int64_t tr = slot_to_row[i]; slot_to_row[i] = slot_to_row[j]; slot_to_row[j] = tr;
            const double te = energies[i]; energies[i] = energies[j]; energies[j] = te;
            const int64_t ts = spin_sums[i]; spin_sums[i] = spin_sums[j]; spin_sums[j] = ts;
            ++acc;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_down_sync(kFull, acc, o);
        ties += __shfl_down_sync(kFull, ties, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (acc && accepted) atomicAdd((unsigned long long*)accepted, (unsigned long long)acc);
        if (ties && near_ties) atomicAdd((unsigned long long*)near_ties, (unsigned long long)ties);
    }
    if (row_to_slot) {
        __syncthreads();
        for (int64_t k = threadIdx.x; k < R; k += blockDim.x) row_to_slot[slot_to_row[k]] = (int32_t)k;
    }
}

// the resident kernels' pair decision (rounds.cuh, swap_decide: FP32 fast
// path, exact FP64 within 1e-5 of the decision) over given inputs, so tests
// can drive it with adversarial u right at the FP64 boundary
__global__ void swap_decide_kernel(const double* __restrict__ bd, const double* __restrict__ Ei,
                                   const double* __restrict__ Ej, const double* __restrict__ u, int64_t n,
                                   uint8_t* __restrict__ accept, uint8_t* __restrict__ near) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        bool nr = false;
        accept[t] = swap_decide(bd[t], Ei[t], Ej[t], u[t], nr) ? 1 : 0;
        near[t] = nr ? 1 : 0;
    }
}

int launch_swap_decide(const double* bd, const double* Ei, const double* Ej, const double* u, int64_t n,
                       uint8_t* accept, uint8_t* near, cudaStream_t s) {
    if (n <= 0) return PTMH_OK;
    swap_decide_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(bd, Ei, Ej, u, n, accept,
                                                                                            near);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

// RngStream.uniform / stream_uniform (rng.py:64-96): out[t] = uniform at
// position pos0 + t of one stream.
__global__ void uniforms_kernel(uint64_t seed, uint64_t stream, uint64_t pos0, int64_t n, double* out) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = stream_uniform(seed, stream, pos0 + (uint64_t)t);
}

// execute_swap_round's decisions (tempering.py:68-86) for an explicit pair
// list: pair k = (pi[k], pj[k]) uses SwapRng.pair_uniform(round, k), i.e.
// stream stream_base + k at position round_index (rng.py:113-116).
__global__ void swap_pairs_kernel(const int64_t* __restrict__ pi, const int64_t* __restrict__ pj, int64_t npairs,
                                  const double* __restrict__ betas, const double* __restrict__ energies,
                                  uint64_t seed, int64_t stream_base, int64_t round_index,
                                  uint8_t* __restrict__ accept, int64_t* near_ties) {
    int ties = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < npairs;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = pi[k], j = pj[k];
        const double u = stream_uniform(seed, (uint64_t)(stream_base + k), (uint64_t)round_index);
        const double x = __dmul_rn(__dsub_rn(betas[i], betas[j]), __dsub_rn(energies[i], energies[j]));
        const double prob = swap_logistic(x);
        if (near_tie(u, prob)) ++ties;
        accept[k] = u < prob ? 1 : 0;
    }
    if (ties && near_ties) atomicAdd((unsigned long long*)near_ties, (unsigned long long)ties);
}

// ------------------------------------------------------------ launchers --
int launch_fill(int8_t* spins, int64_t rows, int64_t n, int64_t up_count, uint64_t seed,
                uint64_t stream0, uint64_t pos0, cudaStream_t s) {
    if (rows == 0) return PTMH_OK;
    if (n <= 200 * 1024) {
        if (n > 48 * 1024)
            PTMH_CUDA(cudaFuncSetAttribute(fill_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)n));
        fill_kernel<true><<<(unsigned)rows, 32, (size_t)n, s>>>(spins, rows, n, up_count, seed,
                                                               stream0, pos0);
    } else {
        fill_kernel<false><<<(unsigned)rows, 32, 0, s>>>(spins, rows, n, up_count, seed, stream0, pos0);
    }
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_row_stats(const int8_t* spins, int64_t rows, int64_t L, int64_t* stats, cudaStream_t s) {
    if (rows == 0) return PTMH_OK;
    row_stats_kernel<<<(unsigned)rows, 256, 0, s>>>(spins, L, stats);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_advance(const AdvanceArgs& a, cudaStream_t s) {
    const int64_t n = a.hi - a.lo;
    if (n <= 0 || a.nsteps <= 0) return PTMH_OK;
    const int warps = 4;
    advance_kernel<<<ceil_div(n, warps), 32 * warps, 0, s>>>(a);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_uniforms(uint64_t seed, uint64_t stream, uint64_t pos0, int64_t n, double* out, cudaStream_t s) {
    if (n <= 0) return PTMH_OK;
    uniforms_kernel<<<std::min<int64_t>(ceil_div(n, 256), 4096), 256, 0, s>>>(seed, stream, pos0, n, out);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_swap_pairs(const int64_t* pi, const int64_t* pj, int64_t npairs, const double* betas,
                      const double* energies, uint64_t seed, int64_t stream_base, int64_t round_index,
                      uint8_t* accept, int64_t* near_ties, cudaStream_t s) {
    if (npairs <= 0) return PTMH_OK;
    swap_pairs_kernel<<<std::min<int64_t>(ceil_div(npairs, 256), 1024), 256, 0, s>>>(
        pi, pj, npairs, betas, energies, seed, stream_base, round_index, accept, near_ties);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

int launch_swap(int64_t* slot_to_row, double* energies, int64_t* spin_sums, const double* betas,
                int64_t R, uint64_t seed, int64_t stream_base, int64_t round_index, int64_t first,
                int64_t pair_lo, int64_t pair_hi, int64_t* accepted, int64_t* near_ties,
                int32_t* row_to_slot, cudaStream_t s, const int64_t* stats, double J, double B) {
    swap_kernel<<<1, 1024, 0, s>>>(slot_to_row, energies, spin_sums, betas, R, seed, stream_base,
                                   round_index, first, pair_lo, pair_hi, accepted, near_ties,
                                   row_to_slot, stats, J, B);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

}  // namespace ptmh

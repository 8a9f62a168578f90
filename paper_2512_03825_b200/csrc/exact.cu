// exact.cu -- the reference's random-site chain on the GPU, bit-exact.
//
// Kernels (reference file:line they reproduce):
//   fill_kernel          kernels.py:26-45   exact-count Fisher-Yates init
//   row_stats_kernel     kernels.py:48-59   integer energy / spin-sum accumulators
//   advance_kernel       kernels.py:62-113  random-site MH, incremental E / sum(s)
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

#include "common.cuh"
#include "launchers.cuh"
#include "philox.cuh"

namespace ptmh {

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
    const uint64_t st = (uint64_t)slot;
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
// (u_acc < exp(-beta*dE_c), kernels.py:95-98) and the mask of earlier
// attempts of the same 32-attempt window whose site is the site or one of its
// neighbours (the dependencies phase 2 must respect).
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
};

__global__ void __launch_bounds__(256) draw_kernel(DrawArgs D) {
    const int64_t npad = (D.n + 31) & ~int64_t(31);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t s = tid / npad;
    if (s >= D.nslots) return;  // whole warps (npad % 32 == 0)
    const int64_t a = tid - s * npad;
    const int lane = threadIdx.x & 31;
    const int64_t slot = D.lo + s;
    const int64_t L = D.L;
    const uint64_t p = D.positions[slot] + 2 * (uint64_t)(D.a0 + a);
    const double u_site = stream_uniform(D.seed, (uint64_t)slot, p);
    const double u_acc = stream_uniform(D.seed, (uint64_t)slot, p + 1);
    const int64_t site = (int64_t)__dmul_rn(u_site, (double)(L * L));
    const int64_t r = site / L, c = site - r * L;
    uint32_t accm = 0;
    const double* tb = D.tbl + slot * 10;
#pragma unroll
    for (int q = 0; q < 10; ++q)
        if (D.dcls[q] > 0.0 && u_acc < tb[q]) accm |= 1u << q;
    // conflicts with earlier attempts of the window: a shifted-2x2-bucket
    // filter (two sites at Chebyshev distance <= 1 share one of 4 buckets),
    // exact neighbour test only where the filter fires
    const unsigned lt_mask = (1u << lane) - 1u;
    bool full = (L & 1) || L <= 8;
    unsigned cand = 0xffffffffu;
    if (!full) {
        const int r1 = (int)(r >> 1), c1 = (int)(c >> 1);
        const int r2 = (int)(((r + 1) % L) >> 1), c2 = (int)(((c + 1) % L) >> 1);
        cand = __match_any_sync(0xffffffffu, (r1 << 16) | c1) | __match_any_sync(0xffffffffu, (r2 << 16) | c1) |
               __match_any_sync(0xffffffffu, (r1 << 16) | c2) | __match_any_sync(0xffffffffu, (r2 << 16) | c2);
    }
    cand &= lt_mask;
    unsigned conf = 0;
    if (__any_sync(0xffffffffu, cand != 0)) {
        const int64_t up = ((r + 1) % L) * L + c, dn = ((r - 1 + L) % L) * L + c;
        const int64_t rt = r * L + (c + 1) % L, lf = r * L + (c - 1 + L) % L;
#pragma unroll 4
        for (int k = 0; k < 32; ++k) {
            const int64_t s2 = __shfl_sync(0xffffffffu, site, k);
            const bool hit = (s2 == site) | (s2 == up) | (s2 == dn) | (s2 == rt) | (s2 == lf);
            conf |= (hit && ((cand >> k) & 1u)) ? (1u << k) : 0u;
        }
    }
    if (a < D.n) {
        const int64_t o = s * D.stride + a;
        D.rec_site[o] = (int32_t)site;
        D.rec_acc[o] = accm;
        D.rec_conf[o] = conf;
    }
}

// Phase 2: warp per slot, windows of 32 attempts committed in dependency
// levels from the phase-1 records; energies summed in attempt order exactly
// as advance_kernel does.
struct CommitArgs {
    AdvanceArgs A;
    int64_t a0, n, stride;
    const int32_t* rec_site;
    const uint32_t* rec_acc;
    const uint32_t* rec_conf;
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
    // spin (+1/-1) at site x; flip of site x
    auto spin = [&](int64_t x) -> int {
        if (kBits) return 2 * (int)((latw[x >> 5] >> (x & 31)) & 1u) - 1;
        return lat[x];
    };
    double e = A.energies[slot];
    long long ssum = A.spin_sums[slot];
    const double nsd = (double)n_sites;
    double acc_d = -0.0;  // int_energy && record == 0: per-lane partial sums (-0.0: identity)
    long long acc_ds = 0;
    const int32_t* rs = C.rec_site + s * C.stride;
    const uint32_t* ra = C.rec_acc + s * C.stride;
    const uint32_t* rc = C.rec_conf + s * C.stride;
    // software pipeline: window w+1's records are loaded, and its lattice
    // lines prefetched into L1, while window w commits (records never depend
    // on the state; a prefetch never changes what a later load returns)
    auto prefetch_site = [&](int64_t st) {
        const int64_t r = st / L, c = st - r * L;
        const int64_t xs[3] = {st, ((r + 1) % L) * L + c, ((r - 1 + L) % L) * L + c};
        for (int q = 0; q < 3; ++q) {
            if (kBits)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(latw + (xs[q] >> 5)));
            else
                asm volatile("prefetch.global.L1 [%0];" ::"l"(lat + xs[q]));
        }
    };
    int64_t n_site = 0;
    uint32_t n_acc = 0u, n_conf = 0u;
    if (lane < C.n) {
        n_site = rs[lane];
        n_acc = ra[lane];
        n_conf = rc[lane];
        prefetch_site(n_site);
    }
    for (int64_t w0 = 0; w0 < C.n; w0 += 32) {
        const int64_t a = w0 + lane;
        const bool valid = a < C.n;
        const int nvalid = (int)min((int64_t)32, C.n - w0);
        const int64_t site = valid ? n_site : 0;
        const uint32_t accm = valid ? n_acc : 0u;
        const unsigned conf = valid ? n_conf : 0u;
        if (a + 32 < C.n) {
            n_site = rs[a + 32];
            n_acc = ra[a + 32];
            n_conf = rc[a + 32];
            prefetch_site(n_site);
        }
        const int64_t r = site / L, c = site - r * L;
        const int64_t up = ((r + 1) % L) * L + c, dn = ((r - 1 + L) % L) * L + c;
        const int64_t rt = r * L + (c + 1) % L, lf = r * L + (c - 1 + L) % L;
        unsigned pending = __ballot_sync(0xffffffffu, valid);
        double my_d = -0.0;  // IEEE identity: keeps a reference -0.0 energy intact
        int my_ds = 0;
        bool my_acc = false;
        while (pending) {
            const bool ready = ((pending >> lane) & 1u) && ((conf & pending) == 0u);
            if (ready) {
                const int sp = spin(site);
                const int nb = spin(up) + spin(dn) + spin(rt) + spin(lf);
                const int cls = (sp > 0 ? 5 : 0) + (nb + 4) / 2;
                const double d = A.dcls[cls];
                if ((d <= 0.0) || ((accm >> cls) & 1u)) {
                    if (kBits)  // lanes of one level may flip different bits of one word
                        atomicXor(&latw[site >> 5], 1u << (site & 31));
                    else
                        lat[site] = (int8_t)(-sp);
                    my_d = d;
                    my_ds = -2 * sp;
                    my_acc = true;
                }
            }
            __syncwarp();
            pending &= ~__ballot_sync(0xffffffffu, ready);
        }
        if (A.int_energy && A.record == 0) {
            // integer increments, nothing recorded: order-free per-lane sums,
            // reduced once after the last window
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
    if (A.int_energy && A.record == 0) {
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

int64_t advance_chunk(int64_t nslots) {
    // attempts per slot per phase-1/phase-2 pass: ~16M records (192 MiB)
    int64_t c = (int64_t(1) << 24) / std::max<int64_t>(1, nslots);
    c = std::max<int64_t>(1024, std::min<int64_t>(c, 1 << 16));
    return c & ~int64_t(31);
}

int64_t advance_ws_bytes(int64_t nslots, int64_t nsteps) {
    const int64_t stride = std::min(advance_chunk(nslots), (nsteps + 31) & ~int64_t(31));
    return nslots * stride * 12;
}

int launch_advance_2phase(const AdvanceArgs& a, void* ws, int64_t ws_bytes, cudaStream_t s) {
    const int64_t nslots = a.hi - a.lo;
    if (nslots <= 0 || a.nsteps <= 0) return PTMH_OK;
    const int64_t stride = std::min(advance_chunk(nslots), (a.nsteps + 31) & ~int64_t(31));
    if (ws_bytes < nslots * stride * 12) {
        set_error("advance workspace too small");
        return PTMH_ERR_ARG;
    }
    int32_t* rs = static_cast<int32_t*>(ws);
    uint32_t* ra = reinterpret_cast<uint32_t*>(rs + nslots * stride);
    uint32_t* rc = ra + nslots * stride;
    for (int64_t a0 = 0; a0 < a.nsteps; a0 += stride) {
        const int64_t n = std::min(stride, a.nsteps - a0);
        DrawArgs D{a.lo, nslots, a.L, a.tbl, a.dcls, a.seed, a.positions, a0, n, stride, rs, ra, rc};
        const int64_t npad = (n + 31) & ~int64_t(31);
        draw_kernel<<<ceil_div(nslots * npad, 256), 256, 0, s>>>(D);
        PTMH_LAUNCH_CHECK();
        CommitArgs C{a, a0, n, stride, rs, ra, rc, a0 + n >= a.nsteps};
        if (a.bits)
            commit_kernel<true><<<ceil_div(nslots, 4), 128, 0, s>>>(C);
        else
            commit_kernel<false><<<ceil_div(nslots, 4), 128, 0, s>>>(C);
        PTMH_LAUNCH_CHECK();
    }
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
__global__ void swap_kernel(int64_t* __restrict__ slot_to_row, double* __restrict__ energies,
                            int64_t* __restrict__ spin_sums, const double* __restrict__ betas,
                            int64_t R, uint64_t seed, int64_t stream_base, int64_t round_index,
                            int64_t first, int64_t pair_lo, int64_t pair_hi,
                            int64_t* accepted, int64_t* near_ties, int32_t* row_to_slot) {
    int acc = 0, ties = 0;
    for (int64_t p = pair_lo + threadIdx.x; p < pair_hi; p += blockDim.x) {
        const int64_t i = first + 2 * p, j = i + 1;
        const double u = stream_uniform(seed, (uint64_t)(stream_base + p), (uint64_t)round_index);
        const double x = __dmul_rn(__dsub_rn(betas[i], betas[j]), __dsub_rn(energies[i], energies[j]));
        double prob;
        if (x >= 0.0) {
            prob = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));
        } else {
            const double ex = exp(x);
            prob = __ddiv_rn(ex, __dadd_rn(1.0, ex));
        }
        // device exp and host libm may differ in the last ulp: count decisions
        // that such a difference could flip (expected: none)
        if (fabs(u - prob) <= 4.0 * 2.220446049250313e-16 * fmax(prob, 2.2250738585072014e-308)) ++ties;
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

int launch_swap(int64_t* slot_to_row, double* energies, int64_t* spin_sums, const double* betas,
                int64_t R, uint64_t seed, int64_t stream_base, int64_t round_index, int64_t first,
                int64_t pair_lo, int64_t pair_hi, int64_t* accepted, int64_t* near_ties,
                int32_t* row_to_slot, cudaStream_t s) {
    swap_kernel<<<1, 1024, 0, s>>>(slot_to_row, energies, spin_sums, betas, R, seed, stream_base,
                                   round_index, first, pair_lo, pair_hi, accepted, near_ties,
                                   row_to_slot);
    PTMH_LAUNCH_CHECK();
    return PTMH_OK;
}

}  // namespace ptmh

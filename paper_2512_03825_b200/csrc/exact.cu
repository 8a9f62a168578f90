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
        double my_d = 0.0;
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

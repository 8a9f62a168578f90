// capi.cu -- extern "C" entry points declared in include/ptmh.h.
//
// (B) device-resident wrappers forward to the launchers in exact.cu /
// checkerboard.cu.  (A) host-buffer entry points reproduce the reference's
// kernel boundary (isingpt/kernels.py) on caller-owned host arrays: they
// stage the arrays in a grow-only device workspace, launch, and copy back.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "launchers.cuh"

namespace ptmh {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

// ------------------------------------------------- host-side table builders --
// dE per class written as the reference writes it (kernels.py:94), and the
// acceptance exponentials with the host libm exp (kernels.py:98).
static double class_delta(int cls, double J, double B) {
    const double s = cls >= 5 ? 1.0 : -1.0;
    const double nb = (double)(2 * (cls % 5) - 4);
    return 2.0 * s * (J * nb - B);
}

static void exact_tables(const double* betas, int64_t R, double J, double B, std::vector<double>& tbl,
                         std::vector<double>& dcls) {
    dcls.resize(10);
    tbl.assign((size_t)R * 10, 1.0);
    for (int c = 0; c < 10; ++c) dcls[c] = class_delta(c, J, B);
    for (int64_t k = 0; k < R; ++k)
        for (int c = 0; c < 10; ++c)
            if (dcls[c] > 0.0) tbl[(size_t)k * 10 + c] = std::exp(-betas[k] * dcls[c]);
}

static uint32_t cb_tables(const double* betas, int64_t R, double J, double B, std::vector<uint32_t>& thr) {
    uint32_t always = 0;
    thr.assign((size_t)R * 10, 0xffffffffu);
    for (int c = 0; c < 10; ++c) {
        const double d = class_delta(c, J, B);
        if (d < 0.0) {
            always |= 1u << c;
            continue;
        }
        if (d == 0.0) {  // neutral: probability 1/2
            for (int64_t k = 0; k < R; ++k) thr[(size_t)k * 10 + c] = 0x80000000u;
            continue;
        }
        for (int64_t k = 0; k < R; ++k) {
            const double p = std::exp(-betas[k] * d);
            const double x = p * 4294967296.0;
            thr[(size_t)k * 10 + c] = x >= 4294967295.0 ? 0xffffffffu : (uint32_t)x;
        }
    }
    if (B == 0.0) always |= 1u << 16;  // thresholds depend on k only
    return always;
}

static bool integral(double x) { return std::isfinite(x) && std::fabs(x) < 1e15 && x == std::floor(x); }

// --------------------------------------------------------------- workspace --
struct Buf {
    void* p = nullptr;
    size_t n = 0;
};

constexpr int kComputeStreams = 4;

struct Workspace {
    std::mutex mu;
    int device = -1;
    std::vector<Buf> bufs;
    cudaStream_t s[3] = {nullptr, nullptr, nullptr};
    cudaStream_t cs[kComputeStreams] = {};  // concurrent chunk compute
    cudaEvent_t ev_in[64], ev_out[64];  // >= chunks per pipelined call
    cudaEvent_t ev_t0, ev_tab;
    bool events = false;
    void* pin = nullptr;  // pinned staging of the small per-call arrays (one H2D, one D2H)
    size_t pin_n = 0;
    bool dirty = false;  // a call returned before its final synchronize (error): drain first
};

// one workspace per device (buffers, streams and events are device-bound),
// each behind its own mutex; created on first use, kept for the process
static std::mutex g_ws_registry_mu;
static std::vector<std::unique_ptr<Workspace>> g_ws_registry;

static int device_workspace(Workspace** out) {
    int dev = 0;
    PTMH_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_ws_registry_mu);
    if ((int)g_ws_registry.size() <= dev) g_ws_registry.resize(dev + 1);
    if (!g_ws_registry[dev]) {
        g_ws_registry[dev].reset(new Workspace());
        g_ws_registry[dev]->device = dev;
    }
    *out = g_ws_registry[dev].get();
    return PTMH_OK;
}

static int ws_prepare(Workspace& w) {
    if (w.dirty) {
        // the previous call failed with work in flight: its copies and kernels
        // (also those on the exact chain's draw/commit side streams, exact.cu)
        // may still use the buffers -- drain the whole device
        cudaDeviceSynchronize();
        cudaGetLastError();
    }
    w.dirty = true;  // cleared by the call's final synchronize
    for (auto& st : w.s)
        if (!st) PTMH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (auto& st : w.cs)
        if (!st) PTMH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    if (!w.events) {
        for (int k = 0; k < 64; ++k) {
            const unsigned fl = getenv("PTMH_TRACE") ? cudaEventDefault : cudaEventDisableTiming;
            PTMH_CUDA(cudaEventCreateWithFlags(&w.ev_in[k], fl));
            PTMH_CUDA(cudaEventCreateWithFlags(&w.ev_out[k], fl));
        }
        PTMH_CUDA(cudaEventCreate(&w.ev_t0));
        PTMH_CUDA(cudaEventCreateWithFlags(&w.ev_tab, cudaEventDisableTiming));
        w.events = true;
    }
    return PTMH_OK;
}

static int ws_pinned(Workspace& w, size_t bytes, uint8_t** out) {
    if (w.pin_n < bytes) {
        if (w.pin) PTMH_CUDA(cudaFreeHost(w.pin));
        w.pin = nullptr;
        w.pin_n = 0;
        PTMH_CUDA(cudaMallocHost(&w.pin, bytes));
        w.pin_n = bytes;
    }
    *out = static_cast<uint8_t*>(w.pin);
    return PTMH_OK;
}

template <typename T>
static int ws_get(Workspace& w, size_t idx, size_t count, T** out) {
    if (w.bufs.size() <= idx) w.bufs.resize(idx + 1);
    Buf& b = w.bufs[idx];
    const size_t bytes = std::max<size_t>(count * sizeof(T), 256);
    if (b.n < bytes) {
        if (b.p) PTMH_CUDA(cudaFree(b.p));
        b.p = nullptr;
        b.n = 0;
        PTMH_CUDA(cudaMalloc(&b.p, bytes));
        b.n = bytes;
    }
    *out = static_cast<T*>(b.p);
    return PTMH_OK;
}

#define PTMH_TRY(expr)          \
    do {                        \
        int rc_ = (expr);       \
        if (rc_ != PTMH_OK) return rc_; \
    } while (0)

}  // namespace ptmh

using namespace ptmh;

extern "C" {

int ptmh_abi_version(void) { return PTMH_ABI_VERSION; }
const char* ptmh_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------- device ABI --
int ptmh_fill_lattices(int8_t* spins, int64_t rows, int64_t L, int64_t up_count, uint64_t seed,
                       uint64_t stream0, uint64_t pos0, void* stream) {
    PTMH_CHECK_ARG(rows >= 0 && L >= 1 && up_count >= 0 && up_count <= L * L, "fill_lattices shape");
    return launch_fill(spins, rows, L * L, up_count, seed, stream0, pos0, as_stream(stream));
}

int64_t ptmh_fill_workspace_bytes(int64_t L, int64_t rows_per_batch) {
    return fill_ws_bytes(L * L, rows_per_batch);
}

int ptmh_fill_lattices_parallel(int8_t* spins, int64_t rows, int64_t L, int64_t up_count, uint64_t seed,
                                uint64_t stream0, uint64_t pos0, void* workspace, int64_t ws_bytes,
                                void* stream) {
    PTMH_CHECK_ARG(rows >= 0 && L >= 1 && up_count >= 0 && up_count <= L * L, "fill_lattices shape");
    return launch_fill_parallel(spins, rows, L * L, up_count, seed, stream0, pos0, workspace, ws_bytes,
                                as_stream(stream));
}

int ptmh_row_stats(const int8_t* spins, int64_t rows, int64_t L, int64_t* stats, void* stream) {
    PTMH_CHECK_ARG(rows >= 0 && L >= 1, "row_stats shape");
    return launch_row_stats(spins, rows, L, stats, as_stream(stream));
}

int ptmh_advance_block(int8_t* spins, int64_t L, const int64_t* slot_to_row, int64_t lo, int64_t hi,
                       const double* tbl, const double* dcls, int int_energy, double* energies,
                       int64_t* spin_sums, uint64_t* positions, int64_t* iters_done, uint64_t seed,
                       int64_t start_iter, int64_t nsteps, double* obs_e, double* obs_m, int64_t ncols,
                       int record, int8_t* states, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L * L < (1LL << 31), "advance_block: need 2 <= L, L*L < 2^31");
    PTMH_CHECK_ARG(lo >= 0 && hi >= lo && nsteps >= 0 && start_iter >= 0, "advance_block range");
    PTMH_CHECK_ARG(record >= 0 && record <= 2, "advance_block record flag");
    PTMH_CHECK_ARG(record == 0 || start_iter + nsteps <= ncols, "advance_block: obs columns");
    AdvanceArgs a{spins, L, slot_to_row, lo, hi, tbl, dcls, int_energy, energies, spin_sums,
                  positions, iters_done, seed, start_iter, nsteps, obs_e, obs_m, ncols, record, states};
    return launch_advance(a, as_stream(stream));
}

int64_t ptmh_advance_workspace_bytes(int64_t nslots, int64_t nsteps) {
    return advance_ws_bytes(nslots, nsteps);
}

int ptmh_advance_block_ws(int8_t* spins, int64_t L, const int64_t* slot_to_row, int64_t lo, int64_t hi,
                          const double* tbl, const double* dcls, int int_energy, double* energies,
                          int64_t* spin_sums, uint64_t* positions, int64_t* iters_done, uint64_t seed,
                          int64_t start_iter, int64_t nsteps, double* obs_e, double* obs_m, int64_t ncols,
                          void* workspace, int64_t ws_bytes, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L <= 4096, "two-phase advance: need 2 <= L <= 4096 (float site rows)");
    PTMH_CHECK_ARG(lo >= 0 && hi >= lo && nsteps >= 0 && start_iter >= 0, "advance_block range");
    PTMH_CHECK_ARG(obs_e == nullptr || start_iter + nsteps <= ncols, "advance_block: obs columns");
    AdvanceArgs a{spins, L, slot_to_row, lo, hi, tbl, dcls, int_energy, energies, spin_sums,
                  positions, iters_done, seed, start_iter, nsteps, obs_e, obs_m, ncols,
                  obs_e ? 1 : 0, nullptr};
    return launch_advance_2phase(a, workspace, ws_bytes, as_stream(stream));
}

int ptmh_bits_pack(const int8_t* spins, int64_t rows, int64_t L, uint32_t* bits, void* stream) {
    PTMH_CHECK_ARG(rows >= 0 && L >= 1, "bits_pack shape");
    return launch_bits_pack(spins, rows, L, bits, as_stream(stream));
}

int ptmh_bits_unpack(const uint32_t* bits, int64_t rows, int64_t L, int8_t* spins, void* stream) {
    PTMH_CHECK_ARG(rows >= 0 && L >= 1, "bits_unpack shape");
    return launch_bits_unpack(bits, rows, L, spins, as_stream(stream));
}

int ptmh_exact_run_resident(uint32_t* bits, int64_t L, int64_t* slot_to_row, int64_t R, const double* tbl,
                            const double* dcls, int int_energy, double* energies, int64_t* spin_sums,
                            uint64_t* positions, int64_t* iters_done, uint64_t seed, int64_t start_iter,
                            int64_t nsteps, int64_t swap_every, int64_t total_iters, const double* betas,
                            int64_t* counters, double* obs_e, double* obs_m, int64_t ncols, void* workspace,
                            int64_t ws_bytes, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L <= 4096 && R >= 1 && R <= 32, "resident exact run: 1 <= R <= 32 slots");
    PTMH_CHECK_ARG(nsteps >= 0 && start_iter >= 1 && swap_every >= 0 && start_iter + nsteps <= total_iters,
                   "resident exact run: iteration range");
    PTMH_CHECK_ARG(obs_e == nullptr || start_iter + nsteps <= ncols, "resident exact run: obs columns");
    AdvanceArgs a{nullptr, L, slot_to_row, 0, R, tbl, dcls, int_energy, energies, spin_sums,
                  positions, iters_done, seed, start_iter, nsteps, obs_e, obs_m, ncols,
                  obs_e ? 1 : 0, nullptr, bits};
    ExactRounds x{swap_every, total_iters, betas, counters};
    return launch_advance_2phase(a, workspace, ws_bytes, as_stream(stream), &x);
}

int ptmh_advance_block_bits(uint32_t* bits, int64_t L, const int64_t* slot_to_row, int64_t lo, int64_t hi,
                            const double* tbl, const double* dcls, int int_energy, double* energies,
                            int64_t* spin_sums, uint64_t* positions, int64_t* iters_done, uint64_t seed,
                            int64_t start_iter, int64_t nsteps, double* obs_e, double* obs_m, int64_t ncols,
                            void* workspace, int64_t ws_bytes, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L <= 4096, "two-phase advance: need 2 <= L <= 4096 (float site rows)");
    PTMH_CHECK_ARG(lo >= 0 && hi >= lo && nsteps >= 0 && start_iter >= 0, "advance_block range");
    PTMH_CHECK_ARG(obs_e == nullptr || start_iter + nsteps <= ncols, "advance_block: obs columns");
    AdvanceArgs a{nullptr, L, slot_to_row, lo, hi, tbl, dcls, int_energy, energies, spin_sums,
                  positions, iters_done, seed, start_iter, nsteps, obs_e, obs_m, ncols,
                  obs_e ? 1 : 0, nullptr, bits};
    return launch_advance_2phase(a, workspace, ws_bytes, as_stream(stream));
}

int ptmh_swap_chunk(int64_t* slot_to_row, double* energies, int64_t* spin_sums, const double* betas,
                    int64_t R, uint64_t seed, int64_t stream_base, int64_t round_index, int64_t first,
                    int64_t pair_lo, int64_t pair_hi, int64_t* accepted, int64_t* near_ties,
                    int32_t* row_to_slot, void* stream) {
    PTMH_CHECK_ARG(pair_lo >= 0 && pair_hi >= pair_lo && first + 2 * pair_hi <= R, "swap_chunk pairs");
    return launch_swap(slot_to_row, energies, spin_sums, betas, R, seed, stream_base, round_index, first,
                       pair_lo, pair_hi, accepted, near_ties, row_to_slot, as_stream(stream));
}

int ptmh_cb_exchange(const int64_t* stats_all, int64_t* slot_to_row, int32_t* row_to_slot, int64_t R,
                     double J, double B, const double* betas, uint64_t seed, int64_t round_index,
                     double* energies, int64_t* spin_sums, int64_t* accepted, int64_t* near_ties,
                     void* stream) {
    PTMH_CHECK_ARG(R >= 1 && round_index >= 0, "cb_exchange args");
    const int64_t first = round_index % 2, n_pairs = std::max<int64_t>(0, (R - first) / 2);
    return launch_swap(slot_to_row, energies, spin_sums, betas, R, seed, R, round_index, first, 0, n_pairs,
                       accepted, near_ties, row_to_slot, as_stream(stream), stats_all, J, B);
}

int64_t ptmh_cb_words_per_color(int64_t L) { return cb_words(L); }

int ptmh_cb_pack(const int8_t* spins, int64_t rows, int64_t L, uint32_t* packed, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L % 2 == 0, "checkerboard needs even L");
    return launch_cb_pack(spins, rows, L, packed, as_stream(stream));
}

int ptmh_cb_unpack(const uint32_t* packed, int64_t rows, int64_t L, int8_t* spins, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L % 2 == 0, "checkerboard needs even L");
    return launch_cb_unpack(packed, rows, L, spins, as_stream(stream));
}

int ptmh_cb_sweeps(uint32_t* packed, int64_t rows, int64_t L, const int32_t* row_to_slot,
                   const uint32_t* thresh, uint32_t always_mask, uint64_t seed, int64_t first_sweep,
                   int64_t n_sweeps, int64_t* stats, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L % 2 == 0 && L <= 65536, "checkerboard needs even 2 <= L <= 65536");
    PTMH_CHECK_ARG(first_sweep >= 0 && n_sweeps >= 0 && first_sweep + n_sweeps < (1LL << 31),
                   "checkerboard sweep index must stay below 2^31");
    return launch_cb_sweeps(packed, rows, L, row_to_slot, thresh, always_mask, seed, first_sweep, n_sweeps,
                            stats, as_stream(stream));
}

int64_t ptmh_cb_sync_words(int64_t rows, int64_t L) {
    // ticket, CTAs out, a counter per lattice, and the persistent kernel's
    // band counters: at most L^2 / 16384 bands per lattice (128-thread items
    // of 2-row strips)
    rows = std::max<int64_t>(rows, 0);
    const int64_t bands = (L >= 1024 && L % 512 == 0) ? L * L / 16384 : 0;
    return 2 + rows + rows * bands;
}

int ptmh_cb_sweeps_sync(uint32_t* packed, int64_t rows, int64_t L, const int32_t* row_to_slot,
                        const uint32_t* thresh, uint32_t always_mask, uint64_t seed, int64_t first_sweep,
                        int64_t n_sweeps, int64_t* stats, uint32_t* sync, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L % 2 == 0 && L <= 65536, "checkerboard needs even 2 <= L <= 65536");
    PTMH_CHECK_ARG(first_sweep >= 0 && n_sweeps >= 0 && first_sweep + n_sweeps < (1LL << 31),
                   "checkerboard sweep index must stay below 2^31");
    return launch_cb_sweeps(packed, rows, L, row_to_slot, thresh, always_mask, seed, first_sweep, n_sweeps,
                            stats, as_stream(stream), sync);
}

int ptmh_cb_sweeps_ws(uint32_t* packed, int64_t rows, int64_t L, const int32_t* row_to_slot,
                      const uint32_t* thresh, uint32_t always_mask, uint64_t seed, int64_t first_sweep,
                      int64_t n_sweeps, int64_t* stats, uint32_t* sync, uint32_t* scratch, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L % 2 == 0 && L <= 65536, "checkerboard needs even 2 <= L <= 65536");
    PTMH_CHECK_ARG(first_sweep >= 0 && n_sweeps >= 0 && first_sweep + n_sweeps < (1LL << 31),
                   "checkerboard sweep index must stay below 2^31");
    PTMH_CHECK_ARG(scratch == nullptr || sync != nullptr, "the scratch buffer needs a sync block");
    return launch_cb_sweeps(packed, rows, L, row_to_slot, thresh, always_mask, seed, first_sweep, n_sweeps,
                            stats, as_stream(stream), sync, scratch);
}

static int run_resident_impl(uint32_t* packed, int64_t R, int64_t L, int64_t* slot_to_row2,
                             int32_t* row_to_slot2, int buf, const uint32_t* thresh, uint32_t always_mask,
                             uint64_t seed, double J, double B, const double* betas, int64_t* stats,
                             int64_t* slot_stats, int64_t* counters, double* obs_e, double* obs_m, int64_t ncols,
                             int64_t first_sweep, int64_t n_sweeps, int64_t total_sweeps, int64_t swap_every,
                             int64_t record_every, int* buf_out, void* stream, int64_t R_total, int rank,
                             int world, int64_t row_lo, int64_t* const* pub_peers, uint32_t* const* flag_peers,
                             int max_ctas, void* ws = nullptr, int64_t ws_bytes = 0) {
    PTMH_CHECK_ARG(L >= 2 && L % 2 == 0 && L <= 65536 && R >= 1 && R < (1LL << 26), "resident shape");
    PTMH_CHECK_ARG(buf == 0 || buf == 1, "resident buffer index");
    PTMH_CHECK_ARG(slot_stats != nullptr || swap_every == 0, "resident slot_stats scratch");
    PTMH_CHECK_ARG(first_sweep >= 0 && n_sweeps >= 0 && first_sweep + n_sweeps <= total_sweeps &&
                       total_sweeps < (1LL << 31), "resident sweep range");
    PTMH_CHECK_ARG(record_every == 0 || (obs_e && obs_m && total_sweeps / record_every <= ncols),
                   "resident observables");
    PTMH_CHECK_ARG(world >= 1 && world <= 8 && rank >= 0 && rank < world && R_total >= R && row_lo >= 0 &&
                       row_lo + R <= R_total, "resident sharding");
    ResidentArgs a{};
    a.packed = packed;
    a.R = (int)R;
    a.L = (int)L;
    a.W = (int)cb_words(L);
    a.WR = (L % 64 == 0) ? (int)(L / 64) : 0;
    a.thresh = thresh;
    a.rk = make_round_keys32(seed);
    a.seed = seed;
    a.J = J;
    a.B = B;
    a.betas = betas;
    a.s2r[0] = slot_to_row2;
    a.s2r[1] = slot_to_row2 + R_total;
    a.r2s[0] = row_to_slot2;
    a.r2s[1] = row_to_slot2 + R;
    a.stats = stats;
    a.slot_stats = slot_stats;
    a.counters = counters;
    a.obs_e = obs_e;
    a.obs_m = obs_m;
    a.ncols = ncols;
    a.first_sweep = first_sweep;
    a.n_sweeps = n_sweeps;
    a.total_sweeps = total_sweeps;
    a.swap_every = swap_every;
    a.record_every = record_every;
    a.buf = buf;
    a.world = world;
    a.rank = rank;
    a.R_total = (int)R_total;
    a.row_lo = row_lo;
    a.max_ctas = max_ctas;
    for (int g = 0; g < world && world > 1; ++g) {
        PTMH_CHECK_ARG(pub_peers && flag_peers && pub_peers[g] && flag_peers[g], "resident peer buffers");
        a.pub_peer[g] = pub_peers[g];
        a.flag_peer[g] = flag_peers[g];
    }
    fill_class_plan(always_mask, &a.n_up, a.up_k, a.up_sf, a.up_cls, &a.ferro);
    int rounds = 0;
    for (int64_t d = first_sweep + 1; d <= first_sweep + n_sweeps; ++d)
        if (swap_every > 0 && d % swap_every == 0 && d < total_sweeps) ++rounds;
    if (buf_out) *buf_out = buf ^ (rounds & 1);
    if (n_sweeps == 0) return PTMH_OK;
    if (ws && swap_every > 0 && rounds > 0 && ws_bytes >= resident_ws_bytes(R_total, rounds) &&
        R_total < (1LL << 24)) {
        a.u_table = static_cast<const double*>(ws);
        a.u_round0 = (first_sweep + swap_every) / swap_every - 1;  // the segment's first round
        a.u_stride = R_total / 2 + 1;
    }
    return launch_cb_resident(a, a.WR > 0, as_stream(stream), nullptr);
}

int ptmh_cb_run_resident(uint32_t* packed, int64_t R, int64_t L, int64_t* slot_to_row2, int32_t* row_to_slot2,
                         int buf, const uint32_t* thresh, uint32_t always_mask, uint64_t seed, double J, double B,
                         const double* betas, int64_t* stats, int64_t* slot_stats, int64_t* counters,
                         double* obs_e, double* obs_m, int64_t ncols, int64_t first_sweep, int64_t n_sweeps,
                         int64_t total_sweeps,
                         int64_t swap_every, int64_t record_every, int* buf_out, void* stream) {
    return run_resident_impl(packed, R, L, slot_to_row2, row_to_slot2, buf, thresh, always_mask, seed, J, B, betas,
                             stats, slot_stats, counters, obs_e, obs_m, ncols, first_sweep, n_sweeps, total_sweeps,
                             swap_every, record_every, buf_out, stream, R, 0, 1, 0, nullptr, nullptr, 0);
}

int64_t ptmh_cb_resident_ws_bytes(int64_t R, int64_t n_rounds) { return resident_ws_bytes(R, n_rounds); }

int ptmh_cb_run_resident_ws(uint32_t* packed, int64_t R, int64_t L, int64_t* slot_to_row2, int32_t* row_to_slot2,
                            int buf, const uint32_t* thresh, uint32_t always_mask, uint64_t seed, double J, double B,
                            const double* betas, int64_t* stats, int64_t* slot_stats, int64_t* counters,
                            double* obs_e, double* obs_m, int64_t ncols, int64_t first_sweep, int64_t n_sweeps,
                            int64_t total_sweeps, int64_t swap_every, int64_t record_every, int* buf_out,
                            void* ws, int64_t ws_bytes, void* stream) {
    return run_resident_impl(packed, R, L, slot_to_row2, row_to_slot2, buf, thresh, always_mask, seed, J, B, betas,
                             stats, slot_stats, counters, obs_e, obs_m, ncols, first_sweep, n_sweeps, total_sweeps,
                             swap_every, record_every, buf_out, stream, R, 0, 1, 0, nullptr, nullptr, 0, ws,
                             ws_bytes);
}

int ptmh_cb_run_resident_sharded_ws(uint32_t* packed, int64_t rows, int64_t L, int64_t* slot_to_row2,
                                    int32_t* row_to_slot2, int buf, const uint32_t* thresh, uint32_t always_mask,
                                    uint64_t seed, double J, double B, const double* betas, int64_t* stats,
                                    int64_t* slot_stats, int64_t* counters, double* obs_e, double* obs_m,
                                    int64_t ncols, int64_t first_sweep, int64_t n_sweeps, int64_t total_sweeps,
                                    int64_t swap_every, int64_t record_every, int* buf_out, int64_t R_total,
                                    int rank, int world, int64_t row_lo, int64_t* const* pub_peers,
                                    uint32_t* const* flag_peers, int max_ctas, void* ws, int64_t ws_bytes,
                                    void* stream) {
    return run_resident_impl(packed, rows, L, slot_to_row2, row_to_slot2, buf, thresh, always_mask, seed, J, B,
                             betas, stats, slot_stats, counters, obs_e, obs_m, ncols, first_sweep, n_sweeps,
                             total_sweeps, swap_every, record_every, buf_out, stream, R_total, rank, world, row_lo,
                             pub_peers, flag_peers, max_ctas, ws, ws_bytes);
}

int ptmh_cb_run_resident_sharded(uint32_t* packed, int64_t rows, int64_t L, int64_t* slot_to_row2,
                                 int32_t* row_to_slot2, int buf, const uint32_t* thresh, uint32_t always_mask,
                                 uint64_t seed, double J, double B, const double* betas, int64_t* stats,
                                 int64_t* slot_stats, int64_t* counters, double* obs_e, double* obs_m,
                                 int64_t ncols, int64_t first_sweep, int64_t n_sweeps, int64_t total_sweeps,
                                 int64_t swap_every, int64_t record_every, int* buf_out, int64_t R_total,
                                 int rank, int world, int64_t row_lo, int64_t* const* pub_peers,
                                 uint32_t* const* flag_peers, int max_ctas, void* stream) {
    return run_resident_impl(packed, rows, L, slot_to_row2, row_to_slot2, buf, thresh, always_mask, seed, J, B,
                             betas, stats, slot_stats, counters, obs_e, obs_m, ncols, first_sweep, n_sweeps,
                             total_sweeps, swap_every, record_every, buf_out, stream, R_total, rank, world, row_lo,
                             pub_peers, flag_peers, max_ctas);
}

// CUDA IPC (one process per GPU): a device allocation's handle, opened as a
// peer pointer by the other ranks (NVLink peer memory for the resident
// kernel's round exchange).
int ptmh_ipc_handle(void* dev_ptr, void* handle_out) {
    PTMH_CHECK_ARG(dev_ptr && handle_out, "ipc handle");
    cudaIpcMemHandle_t h;
    PTMH_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
    std::memcpy(handle_out, &h, sizeof(h));
    return PTMH_OK;
}

int ptmh_ipc_open(const void* handle, void** dev_ptr_out) {
    PTMH_CHECK_ARG(handle && dev_ptr_out, "ipc open");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    PTMH_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    return PTMH_OK;
}

int ptmh_ipc_close(void* dev_ptr) {
    PTMH_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return PTMH_OK;
}

int64_t ptmh_ipc_handle_bytes(void) { return (int64_t)sizeof(cudaIpcMemHandle_t); }

// A dedicated, zeroed device allocation for buffers shared over IPC: a handle
// names a whole cudaMalloc allocation, so a sub-block of a caching allocator's
// segment (a torch tensor) would be opened at the segment's base.
int ptmh_peer_alloc(int64_t bytes, void** dev_ptr_out) {
    PTMH_CHECK_ARG(bytes > 0 && dev_ptr_out, "peer alloc");
    PTMH_CUDA(cudaMalloc(dev_ptr_out, (size_t)bytes));
    PTMH_CUDA(cudaMemset(*dev_ptr_out, 0, (size_t)bytes));
    return PTMH_OK;
}

int ptmh_peer_free(void* dev_ptr) {
    PTMH_CUDA(cudaFree(dev_ptr));
    return PTMH_OK;
}

int ptmh_cb_unpack_slots(const uint32_t* packed, const int64_t* slot_to_row, int64_t R, int64_t L,
                         int8_t* out, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L % 2 == 0 && R >= 0, "cb_unpack_slots shape");
    return launch_cb_unpack_slots(packed, slot_to_row, R, L, out, as_stream(stream));
}

int ptmh_cb_row_stats(const uint32_t* packed, int64_t rows, int64_t L, int64_t* stats, void* stream) {
    PTMH_CHECK_ARG(L >= 2 && L % 2 == 0, "checkerboard needs even L");
    return launch_cb_row_stats(packed, rows, L, stats, as_stream(stream));
}

int ptmh_cb_slot_energies(const int64_t* stats_all, const int64_t* slot_to_row, int64_t R, double J, double B,
                          double* energies, int64_t* spin_sums, void* stream) {
    return launch_cb_slot_energies(stats_all, slot_to_row, R, J, B, energies, spin_sums, as_stream(stream));
}

int ptmh_cb_observe(const int64_t* stats_all, const int64_t* slot_to_row, int64_t R, int64_t L, double J,
                    double B, double* obs_e, double* obs_m, int64_t ncols, int64_t col, void* stream) {
    PTMH_CHECK_ARG(col >= 0 && col < ncols, "observe column");
    return launch_cb_observe(stats_all, slot_to_row, R, L, J, B, obs_e, obs_m, ncols, col, as_stream(stream));
}

int ptmh_cb_last_launch(int32_t* info) {
    PTMH_CHECK_ARG(info, "cb_last_launch out");
    const CbLaunchInfo c = cb_last_launch();
    const int32_t v[6] = {c.kind, c.rows, c.threads, c.group, c.bands, c.grid};
    std::memcpy(info, v, sizeof(v));
    return PTMH_OK;
}

int ptmh_uniforms(uint64_t seed, uint64_t stream_id, uint64_t position, int64_t n, double* out, void* stream) {
    PTMH_CHECK_ARG(n >= 0, "uniforms count");
    return launch_uniforms(seed, stream_id, position, n, out, as_stream(stream));
}

// --------------------------------------------------------------- host ABI --
int ptmh_host_fill_lattice(int8_t* out, int64_t n, int64_t up_count, uint64_t seed, uint64_t stream,
                           uint64_t position, uint64_t* new_position) {
    PTMH_CHECK_ARG(n >= 1 && up_count >= 0, "fill_lattice shape");
    Workspace* wsp = nullptr;
    PTMH_TRY(device_workspace(&wsp));
    Workspace& g_ws = *wsp;
    std::lock_guard<std::mutex> lk(g_ws.mu);
    PTMH_TRY(ws_prepare(g_ws));
    cudaStream_t s = g_ws.s[1];
    int8_t* d = nullptr;
    PTMH_TRY(ws_get(g_ws, 0, (size_t)n, &d));
    PTMH_TRY(launch_fill(d, 1, n, up_count, seed, stream, position, s));
    PTMH_CUDA(cudaMemcpyAsync(out, d, (size_t)n, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaStreamSynchronize(s));
    g_ws.dirty = false;
    if (new_position) *new_position = position + (uint64_t)(n - 1);  // kernels.py:45
    return PTMH_OK;
}

int ptmh_host_lattice_energy(const int8_t* spins, int64_t L, double J, double B, double* energy) {
    PTMH_CHECK_ARG(L >= 1 && energy, "lattice_energy shape");
    Workspace* wsp = nullptr;
    PTMH_TRY(device_workspace(&wsp));
    Workspace& g_ws = *wsp;
    std::lock_guard<std::mutex> lk(g_ws.mu);
    PTMH_TRY(ws_prepare(g_ws));
    cudaStream_t s = g_ws.s[1];
    int8_t* d = nullptr;
    int64_t* st = nullptr;
    PTMH_TRY(ws_get(g_ws, 0, (size_t)(L * L), &d));
    PTMH_TRY(ws_get(g_ws, 1, 2, &st));
    int64_t h[2];
    PTMH_CUDA(cudaMemcpyAsync(d, spins, (size_t)(L * L), cudaMemcpyHostToDevice, s));
    PTMH_TRY(launch_row_stats(d, 1, L, st, s));
    PTMH_CUDA(cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaStreamSynchronize(s));
    g_ws.dirty = false;
    *energy = B * (double)h[0] - J * (double)h[1];  // kernels.py:59
    return PTMH_OK;
}

int ptmh_host_advance_block(int8_t* spins, int64_t rows, int64_t L, const int64_t* slot_to_row, int64_t R,
                            int64_t lo, int64_t hi, const double* betas, double J, double B,
                            double* energies, int64_t* spin_sums, uint64_t* positions,
                            int64_t* iters_done, uint64_t seed, int64_t start_iter, int64_t nsteps,
                            double* obs_e, double* obs_m, int64_t ncols, int record, int8_t* states) {
    PTMH_CHECK_ARG(rows >= 1 && R >= 1 && lo >= 0 && hi <= R && lo <= hi, "advance_block shape");
    PTMH_CHECK_ARG(record == 0 || (obs_e && obs_m && start_iter + nsteps <= ncols), "advance_block obs");
    PTMH_CHECK_ARG(record != 2 || states, "advance_block states");
    if (hi == lo || nsteps == 0) {
        for (int64_t k = lo; k < hi; ++k) iters_done[k] = start_iter + nsteps;
        return PTMH_OK;
    }
    std::vector<double> tbl, dcls;
    exact_tables(betas, R, J, B, tbl, dcls);
    int int_energy = integral(J) && integral(B) && std::fabs(J) <= 1e6 && std::fabs(B) <= 1e6;
    for (int64_t k = lo; k < hi && int_energy; ++k) int_energy = integral(energies[k]);
    Workspace* wsp = nullptr;
    PTMH_TRY(device_workspace(&wsp));
    Workspace& g_ws = *wsp;
    std::lock_guard<std::mutex> lk(g_ws.mu);
    PTMH_TRY(ws_prepare(g_ws));
    cudaStream_t s = g_ws.s[1];
    const size_t nsite = (size_t)(L * L);
    int8_t* d_spins; int64_t* d_s2r; double *d_tbl, *d_dcls, *d_e, *d_oe = nullptr, *d_om = nullptr;
    int64_t *d_sums, *d_iters; uint64_t* d_pos; int8_t* d_states = nullptr;
    PTMH_TRY(ws_get(g_ws, 0, (size_t)rows * nsite, &d_spins));
    PTMH_TRY(ws_get(g_ws, 1, (size_t)R, &d_s2r));
    PTMH_TRY(ws_get(g_ws, 2, (size_t)R * 10, &d_tbl));
    PTMH_TRY(ws_get(g_ws, 3, 10, &d_dcls));
    PTMH_TRY(ws_get(g_ws, 4, (size_t)R, &d_e));
    PTMH_TRY(ws_get(g_ws, 5, (size_t)R, &d_sums));
    PTMH_TRY(ws_get(g_ws, 6, (size_t)R, &d_pos));
    PTMH_TRY(ws_get(g_ws, 7, (size_t)R, &d_iters));
    PTMH_CUDA(cudaMemcpyAsync(d_spins, spins, (size_t)rows * nsite, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_s2r, slot_to_row, R * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_tbl, tbl.data(), R * 80, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_dcls, dcls.data(), 80, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_e, energies, R * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_sums, spin_sums, R * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_pos, positions, R * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_iters, iters_done, R * 8, cudaMemcpyHostToDevice, s));
    if (record >= 1) {
        PTMH_TRY(ws_get(g_ws, 8, (size_t)R * ncols, &d_oe));
        PTMH_TRY(ws_get(g_ws, 9, (size_t)R * ncols, &d_om));
    }
    if (record == 2) PTMH_TRY(ws_get(g_ws, 10, (size_t)R * ncols * nsite, &d_states));
    AdvanceArgs a{d_spins, L, d_s2r, lo, hi, d_tbl, d_dcls, int_energy, d_e, d_sums, d_pos, d_iters, seed,
                  start_iter, nsteps, d_oe, d_om, ncols, record, d_states};
    if (record <= 1 && L <= 4096) {  // bit-packed lattices: L2-resident random-site commits
        const int64_t wsb = advance_ws_bytes(hi - lo, nsteps);
        void* d_ws = nullptr;
        uint32_t* d_bits = nullptr;
        PTMH_TRY(ws_get(g_ws, 17, (size_t)wsb, reinterpret_cast<int8_t**>(&d_ws)));
        PTMH_TRY(ws_get(g_ws, 18, (size_t)rows * (size_t)((nsite + 31) / 32), &d_bits));
        PTMH_TRY(launch_bits_pack(d_spins, rows, L, d_bits, s));
        a.bits = d_bits;
        PTMH_TRY(launch_advance_2phase(a, d_ws, wsb, s));
        PTMH_TRY(launch_bits_unpack(d_bits, rows, L, d_spins, s));
    } else {
        PTMH_TRY(launch_advance(a, s));
    }
    PTMH_CUDA(cudaMemcpyAsync(spins, d_spins, (size_t)rows * nsite, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaMemcpyAsync(energies + lo, d_e + lo, (hi - lo) * 8, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaMemcpyAsync(spin_sums + lo, d_sums + lo, (hi - lo) * 8, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaMemcpyAsync(positions + lo, d_pos + lo, (hi - lo) * 8, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaMemcpyAsync(iters_done + lo, d_iters + lo, (hi - lo) * 8, cudaMemcpyDeviceToHost, s));
    if (record >= 1) {
        // only the columns this call wrote, as the numba kernel does
        const size_t pitch = (size_t)ncols * 8;
        PTMH_CUDA(cudaMemcpy2DAsync(obs_e + lo * ncols + start_iter, pitch, d_oe + lo * ncols + start_iter,
                                    pitch, nsteps * 8, hi - lo, cudaMemcpyDeviceToHost, s));
        PTMH_CUDA(cudaMemcpy2DAsync(obs_m + lo * ncols + start_iter, pitch, d_om + lo * ncols + start_iter,
                                    pitch, nsteps * 8, hi - lo, cudaMemcpyDeviceToHost, s));
    }
    if (record == 2) {
        const size_t pitch = (size_t)ncols * nsite;
        PTMH_CUDA(cudaMemcpy2DAsync(states + (lo * ncols + start_iter) * nsite, pitch,
                                    d_states + (lo * ncols + start_iter) * nsite, pitch, nsteps * nsite,
                                    hi - lo, cudaMemcpyDeviceToHost, s));
    }
    PTMH_CUDA(cudaStreamSynchronize(s));
    g_ws.dirty = false;
    return PTMH_OK;
}

int ptmh_host_swap_chunk(int64_t* slot_to_row, double* energies, int64_t* spin_sums, const double* betas,
                         int64_t R, uint64_t seed, int64_t stream_base, int64_t round_index, int64_t first,
                         int64_t pair_lo, int64_t pair_hi, int64_t* accepted) {
    PTMH_CHECK_ARG(R >= 0 && pair_lo >= 0 && pair_hi >= pair_lo && first + 2 * pair_hi <= R,
                   "swap_chunk pairs");
    if (accepted) *accepted = 0;
    if (pair_hi == pair_lo) return PTMH_OK;
    Workspace* wsp = nullptr;
    PTMH_TRY(device_workspace(&wsp));
    Workspace& g_ws = *wsp;
    std::lock_guard<std::mutex> lk(g_ws.mu);
    PTMH_TRY(ws_prepare(g_ws));
    cudaStream_t s = g_ws.s[1];
    int64_t *d_s2r, *d_sums, *d_cnt; double *d_e, *d_b;
    PTMH_TRY(ws_get(g_ws, 1, (size_t)R, &d_s2r));
    PTMH_TRY(ws_get(g_ws, 4, (size_t)R, &d_e));
    PTMH_TRY(ws_get(g_ws, 5, (size_t)R, &d_sums));
    PTMH_TRY(ws_get(g_ws, 11, (size_t)R, &d_b));
    PTMH_TRY(ws_get(g_ws, 12, 2, &d_cnt));
    PTMH_CUDA(cudaMemcpyAsync(d_s2r, slot_to_row, R * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_e, energies, R * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_sums, spin_sums, R * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_b, betas, R * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemsetAsync(d_cnt, 0, 16, s));
    PTMH_TRY(launch_swap(d_s2r, d_e, d_sums, d_b, R, seed, stream_base, round_index, first, pair_lo, pair_hi,
                         d_cnt, d_cnt + 1, nullptr, s));
    int64_t cnt[2];
    PTMH_CUDA(cudaMemcpyAsync(slot_to_row, d_s2r, R * 8, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaMemcpyAsync(energies, d_e, R * 8, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaMemcpyAsync(spin_sums, d_sums, R * 8, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaMemcpyAsync(cnt, d_cnt, 16, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaStreamSynchronize(s));
    g_ws.dirty = false;
    if (accepted) *accepted = cnt[0];
    return PTMH_OK;
}

// ---- the reference's per-replica public ops (rng.py:64-116, mh.py:73-88,
// tempering.py:68-86) on the device; the Python layer (rng.py, mh.py,
// tempering.py in this package) keeps the reference's objects on the host.
int ptmh_host_uniforms(uint64_t seed, uint64_t stream, uint64_t position, int64_t n, double* out) {
    PTMH_CHECK_ARG(n >= 0 && (n == 0 || out), "uniforms count");
    if (n == 0) return PTMH_OK;
    Workspace* wsp = nullptr;
    PTMH_TRY(device_workspace(&wsp));
    Workspace& g_ws = *wsp;
    std::lock_guard<std::mutex> lk(g_ws.mu);
    PTMH_TRY(ws_prepare(g_ws));
    cudaStream_t s = g_ws.s[1];
    double* d = nullptr;
    PTMH_TRY(ws_get(g_ws, 20, (size_t)n, &d));
    PTMH_TRY(launch_uniforms(seed, stream, position, n, d, s));
    PTMH_CUDA(cudaMemcpyAsync(out, d, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaStreamSynchronize(s));
    g_ws.dirty = false;
    return PTMH_OK;
}

int ptmh_swap_decide(const double* bd, const double* Ei, const double* Ej, const double* u, int64_t n,
                     uint8_t* accept, uint8_t* near, void* stream) {
    PTMH_CHECK_ARG(n >= 0, "swap_decide: n >= 0");
    return launch_swap_decide(bd, Ei, Ej, u, n, accept, near, as_stream(stream));
}

int ptmh_host_swap_pairs(const int64_t* pair_i, const int64_t* pair_j, int64_t npairs, const double* betas,
                         const double* energies, int64_t n, uint64_t seed, int64_t stream_base,
                         int64_t round_index, uint8_t* accept, int64_t* near_ties) {
    PTMH_CHECK_ARG(npairs >= 0 && n >= 0 && stream_base >= 0 && round_index >= 0, "swap_pairs shape");
    for (int64_t k = 0; k < npairs; ++k)
        PTMH_CHECK_ARG(pair_i[k] >= 0 && pair_i[k] < n && pair_j[k] >= 0 && pair_j[k] < n,
                       "swap_pairs index out of range");
    if (near_ties) *near_ties = 0;
    if (npairs == 0) return PTMH_OK;
    Workspace* wsp = nullptr;
    PTMH_TRY(device_workspace(&wsp));
    Workspace& g_ws = *wsp;
    std::lock_guard<std::mutex> lk(g_ws.mu);
    PTMH_TRY(ws_prepare(g_ws));
    cudaStream_t s = g_ws.s[1];
    int64_t *d_i, *d_j, *d_cnt;
    double *d_b, *d_e;
    uint8_t* d_acc;
    PTMH_TRY(ws_get(g_ws, 21, (size_t)npairs, &d_i));
    PTMH_TRY(ws_get(g_ws, 22, (size_t)npairs, &d_j));
    PTMH_TRY(ws_get(g_ws, 23, (size_t)n, &d_b));
    PTMH_TRY(ws_get(g_ws, 24, (size_t)n, &d_e));
    PTMH_TRY(ws_get(g_ws, 25, (size_t)npairs, &d_acc));
    PTMH_TRY(ws_get(g_ws, 26, 1, &d_cnt));
    PTMH_CUDA(cudaMemcpyAsync(d_i, pair_i, npairs * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_j, pair_j, npairs * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_b, betas, n * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemcpyAsync(d_e, energies, n * 8, cudaMemcpyHostToDevice, s));
    PTMH_CUDA(cudaMemsetAsync(d_cnt, 0, 8, s));
    PTMH_TRY(launch_swap_pairs(d_i, d_j, npairs, d_b, d_e, seed, stream_base, round_index, d_acc, d_cnt, s));
    int64_t ties = 0;
    PTMH_CUDA(cudaMemcpyAsync(accept, d_acc, (size_t)npairs, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaMemcpyAsync(&ties, d_cnt, 8, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaStreamSynchronize(s));
    g_ws.dirty = false;
    if (near_ties) *near_ties = ties;
    return PTMH_OK;
}

int ptmh_host_mh_steps(int8_t* spins, int64_t L, double beta, double J, double B, double* energy,
                       int64_t* spin_sum, uint64_t seed, uint64_t stream, uint64_t* position,
                       int64_t nsteps) {
    PTMH_CHECK_ARG(L >= 2 && nsteps >= 0 && energy && spin_sum && position, "mh_steps shape");
    if (nsteps == 0) return PTMH_OK;
    std::vector<double> tbl, dcls;
    exact_tables(&beta, 1, J, B, tbl, dcls);
    const int int_energy = integral(J) && integral(B) && std::fabs(J) <= 1e6 && std::fabs(B) <= 1e6 &&
                           integral(*energy);
    Workspace* wsp = nullptr;
    PTMH_TRY(device_workspace(&wsp));
    Workspace& g_ws = *wsp;
    std::lock_guard<std::mutex> lk(g_ws.mu);
    PTMH_TRY(ws_prepare(g_ws));
    cudaStream_t s = g_ws.s[1];
    const size_t nsite = (size_t)(L * L);
    // one pinned block each way: lattice, table, (row 0, e, sum, pos, iters)
    const size_t small = 5 * 8, tb = 20 * 8, bytes = small + tb + nsite;
    uint8_t* pin = nullptr;
    PTMH_TRY(ws_pinned(g_ws, bytes, &pin));
    int64_t* hs = reinterpret_cast<int64_t*>(pin);
    hs[0] = 0;
    std::memcpy(&hs[1], energy, 8);
    hs[2] = *spin_sum;
    std::memcpy(&hs[3], position, 8);
    hs[4] = 0;
    std::memcpy(pin + small, tbl.data(), 10 * 8);
    std::memcpy(pin + small + 80, dcls.data(), 10 * 8);
    std::memcpy(pin + small + tb, spins, nsite);
    uint8_t* d = nullptr;
    PTMH_TRY(ws_get(g_ws, 27, bytes, &d));
    PTMH_CUDA(cudaMemcpyAsync(d, pin, bytes, cudaMemcpyHostToDevice, s));
    int64_t* ds = reinterpret_cast<int64_t*>(d);
    AdvanceArgs a{reinterpret_cast<int8_t*>(d + small + tb), L, ds, 0, 1,
                  reinterpret_cast<const double*>(d + small), reinterpret_cast<const double*>(d + small + 80),
                  int_energy, reinterpret_cast<double*>(ds + 1), ds + 2, reinterpret_cast<uint64_t*>(ds + 3),
                  ds + 4, seed, 0, nsteps, nullptr, nullptr, 0, 0, nullptr, nullptr, stream};
    PTMH_TRY(launch_advance(a, s));
    PTMH_CUDA(cudaMemcpyAsync(pin, d, bytes, cudaMemcpyDeviceToHost, s));
    PTMH_CUDA(cudaStreamSynchronize(s));
    g_ws.dirty = false;
    std::memcpy(energy, &hs[1], 8);
    *spin_sum = hs[2];
    std::memcpy(position, &hs[3], 8);
    std::memcpy(spins, pin + small + tb, nsite);
    return PTMH_OK;
}

int ptmh_host_cb_interval(int8_t* spins, int64_t R, int64_t L, int64_t* slot_to_row, const double* betas,
                          double J, double B, uint64_t seed, int64_t first_sweep, int64_t n_sweeps,
                          int64_t round_index, double* energies, int64_t* spin_sums, int64_t* accepted) {
    PTMH_CHECK_ARG(R >= 1 && L >= 2 && L % 2 == 0 && L <= 65536, "cb_interval shape");
    PTMH_CHECK_ARG(first_sweep >= 0 && n_sweeps >= 0, "cb_interval sweeps");
    std::vector<uint32_t> thr;
    const uint32_t always = cb_tables(betas, R, J, B, thr);
    std::vector<int32_t> r2s((size_t)R);
    for (int64_t k = 0; k < R; ++k) {
        PTMH_CHECK_ARG(slot_to_row[k] >= 0 && slot_to_row[k] < R, "slot_to_row out of range");
        r2s[(size_t)slot_to_row[k]] = (int32_t)k;
    }
    Workspace* wsp = nullptr;
    PTMH_TRY(device_workspace(&wsp));
    Workspace& g_ws = *wsp;
    std::lock_guard<std::mutex> lk(g_ws.mu);
    PTMH_TRY(ws_prepare(g_ws));
    cudaStream_t sin = g_ws.s[0], sc = g_ws.s[1], sout = g_ws.s[2];
    if (getenv("PTMH_DEBUG")) {
        cudaPointerAttributes pa;
        cudaError_t e = cudaPointerGetAttributes(&pa, spins);
        fprintf(stderr, "ptmh: spins %p attr rc=%d type=%d\n", (void*)spins, (int)e, (int)pa.type);
    }
    const int64_t nsite = L * L, W = cb_words(L);
    int8_t* d_spins;
    uint32_t* d_packed;
    int64_t* d_stats;
    PTMH_TRY(ws_get(g_ws, 0, (size_t)(R * nsite), &d_spins));
    PTMH_TRY(ws_get(g_ws, 13, (size_t)(R * 2 * W), &d_packed));
    PTMH_TRY(ws_get(g_ws, 14, (size_t)(R * 2), &d_stats));
    // The small arrays travel as one block each way (pinned staging, one H2D
    // and one D2H instead of nine copies from pageable memory: 8-byte
    // aligned offsets) -- outputs first: slot_to_row | energies | spin_sums |
    // counters, then the inputs only: betas | thresholds | row_to_slot.
    const size_t o_e = 8 * R, o_sums = 16 * R, o_cnt = 24 * R, o_b = o_cnt + 16, o_thr = o_b + 8 * R,
                 o_r2s = o_thr + 40 * R, n_small = o_r2s + 8 * R, n_out = o_cnt + 16;
    uint8_t *h_small, *d_small;
    PTMH_TRY(ws_pinned(g_ws, n_small, &h_small));
    PTMH_TRY(ws_get(g_ws, 19, n_small, &d_small));
    memcpy(h_small, slot_to_row, 8 * R);
    memset(h_small + o_e, 0, o_b - o_e);  // energies, sums (recomputed on the device), counters = 0
    memcpy(h_small + o_b, betas, 8 * R);
    memcpy(h_small + o_thr, thr.data(), 40 * R);
    memcpy(h_small + o_r2s, r2s.data(), 4 * R);
    int64_t* d_s2r = reinterpret_cast<int64_t*>(d_small);
    double* d_e = reinterpret_cast<double*>(d_small + o_e);
    int64_t* d_sums = reinterpret_cast<int64_t*>(d_small + o_sums);
    int64_t* d_cnt = reinterpret_cast<int64_t*>(d_small + o_cnt);
    double* d_b = reinterpret_cast<double*>(d_small + o_b);
    uint32_t* d_thr = reinterpret_cast<uint32_t*>(d_small + o_thr);
    int32_t* d_r2s = reinterpret_cast<int32_t*>(d_small + o_r2s);
    // Replica chunks pipeline the lattice copies with the compute.  One chunk
    // per 2 MiB of int8 lattices, at most 8 (measured per call: C1 (8 KiB) 1
    // chunk 134 us vs 8: 280 us; C2 (4 MiB) 2: 254 vs 8: 314 us; C5 (16 MiB)
    // 8: 716 us vs 1: 858 us; C3 (256 MiB) 8: 6.6 ms vs 4: 7.1, 16: 6.7).
    const char* pc = getenv("PTMH_PLUGIN_CHUNKS");  // A/B, tools/ only
    const int64_t nch = std::min<int64_t>(
        R, pc ? std::max(1, std::min(64, atoi(pc))) : std::max<int64_t>(1, std::min<int64_t>(8, R * nsite >> 21)));
    uint32_t* d_sync = nullptr;  // one persistent-sweep sync block per chunk
    const int64_t sync_words = ptmh_cb_sync_words(R, L);
    // Chunk compute: where the persistent path applies, every chunk runs on
    // ONE stream as one persistent launch (it fills the GPU by itself; two
    // of them side by side cost 2x, 16.9 vs 7.2 ms per C3 call); otherwise
    // the per-launch kernels of a chunk do not fill the GPU and the chunks run
    // on kComputeStreams concurrent streams.  PTMH_PLUGIN_SYNC=0 forces the
    // latter (A/B, tools/ only).
    const char* ps = getenv("PTMH_PLUGIN_SYNC");
    const bool plugin_sync = !(ps && ps[0] == '0') && cb_sweeps_persistent_applies(L, always, n_sweeps);
    uint32_t* d_scratch = nullptr;  // the temporally blocked persistent path's second state buffer
    if (plugin_sync) {
        PTMH_TRY(ws_get(g_ws, 17, (size_t)(nch * sync_words), &d_sync));
        PTMH_CUDA(cudaMemsetAsync(d_sync, 0, (size_t)(nch * sync_words) * 4, sc));
        PTMH_TRY(ws_get(g_ws, 28, (size_t)(R * 2 * W), &d_scratch));
    }
    auto chunk = [&](int64_t c, int64_t& lo, int64_t& n) {
        lo = R * c / nch;
        n = R * (c + 1) / nch - lo;
    };
    auto compute = [&](int64_t lo, int64_t n, uint32_t* sync, cudaStream_t cst) -> int {
        PTMH_TRY(launch_cb_pack(d_spins + lo * nsite, n, L, d_packed + lo * 2 * W, cst));
        PTMH_TRY(launch_cb_row_stats(d_packed + lo * 2 * W, n, L, d_stats + 2 * lo, cst));
        PTMH_TRY(launch_cb_sweeps(d_packed + lo * 2 * W, n, L, d_r2s + lo, d_thr, always, seed, first_sweep,
                                  n_sweeps, d_stats + 2 * lo, cst, sync,
                                  sync && d_scratch ? d_scratch + lo * 2 * W : nullptr));
        PTMH_TRY(launch_cb_unpack(d_packed + lo * 2 * W, n, L, d_spins + lo * nsite, cst));
        return PTMH_OK;
    };
    if (nch == 1 && !getenv("PTMH_TRACE")) {  // small call: everything in order on one stream
        PTMH_CUDA(cudaMemcpyAsync(d_small, h_small, n_small, cudaMemcpyHostToDevice, sc));
        PTMH_CUDA(cudaMemcpyAsync(d_spins, spins, (size_t)(R * nsite), cudaMemcpyHostToDevice, sc));
        PTMH_TRY(compute(0, R, d_sync, sc));
        PTMH_CUDA(cudaMemcpyAsync(spins, d_spins, (size_t)(R * nsite), cudaMemcpyDeviceToHost, sc));
    } else {
        // pipeline over replica chunks: all H2D copies are issued first, then
        // the compute chain (each chunk waits for its copy), then the D2H
        // copies (each waits for its chunk), so no queue ever blocks behind a
        // later dependency
        // (the small block goes first on the lattice copy queue: the compute
        // streams see it through ev_in, sc through ev_out.  Issued on sc
        // beside the chunk copies instead, a C3 call took 9.3 ms, not 6.6.)
        if (getenv("PTMH_TRACE")) PTMH_CUDA(cudaEventRecord(g_ws.ev_t0, sin));
        PTMH_CUDA(cudaMemcpyAsync(d_small, h_small, n_small, cudaMemcpyHostToDevice, sin));
        for (int64_t c = 0; c < nch; ++c) {
            int64_t lo, n;
            chunk(c, lo, n);
            PTMH_CUDA(cudaMemcpyAsync(d_spins + lo * nsite, spins + lo * nsite, (size_t)(n * nsite),
                                      cudaMemcpyHostToDevice, sin));
            PTMH_CUDA(cudaEventRecord(g_ws.ev_in[c], sin));
        }
        // the sync-block reset is on sc: every compute stream starts after it
        PTMH_CUDA(cudaEventRecord(g_ws.ev_tab, sc));
        for (int64_t c = 0; c < nch; ++c) {
            int64_t lo, n;
            chunk(c, lo, n);
            cudaStream_t cst = plugin_sync ? g_ws.cs[0] : g_ws.cs[c % kComputeStreams];
            PTMH_CUDA(cudaStreamWaitEvent(cst, g_ws.ev_tab, 0));
            PTMH_CUDA(cudaStreamWaitEvent(cst, g_ws.ev_in[c], 0));
            PTMH_TRY(compute(lo, n, plugin_sync ? d_sync + c * sync_words : nullptr, cst));
            PTMH_CUDA(cudaEventRecord(g_ws.ev_out[c], cst));
            PTMH_CUDA(cudaStreamWaitEvent(sc, g_ws.ev_out[c], 0));  // the exchange needs every chunk
        }
        for (int64_t c = 0; c < nch; ++c) {
            int64_t lo, n;
            chunk(c, lo, n);
            PTMH_CUDA(cudaStreamWaitEvent(sout, g_ws.ev_out[c], 0));
            PTMH_CUDA(cudaMemcpyAsync(spins + lo * nsite, d_spins + lo * nsite, (size_t)(n * nsite),
                                      cudaMemcpyDeviceToHost, sout));
        }
        if (getenv("PTMH_TRACE")) {  // per-chunk timeline (tools/ only)
            PTMH_CUDA(cudaStreamSynchronize(sout));
            PTMH_CUDA(cudaStreamSynchronize(sc));
            float t_in = 0, t_out = 0;
            for (int64_t c = 0; c < nch; ++c) {
                PTMH_CUDA(cudaEventElapsedTime(&t_in, g_ws.ev_t0, g_ws.ev_in[c]));
                PTMH_CUDA(cudaEventElapsedTime(&t_out, g_ws.ev_t0, g_ws.ev_out[c]));
                fprintf(stderr, "ptmh trace chunk %ld: h2d done %.3f ms, compute done %.3f ms\n", (long)c, t_in,
                        t_out);
            }
        }
    }
    if (round_index >= 0) {  // energies by slot + the round, one launch
        const int64_t first = round_index % 2, n_pairs = std::max<int64_t>(0, (R - first) / 2);
        PTMH_TRY(launch_swap(d_s2r, d_e, d_sums, d_b, R, seed, R, round_index, first, 0, n_pairs, d_cnt,
                             d_cnt + 1, nullptr, sc, d_stats, J, B));
    } else {
        PTMH_TRY(launch_cb_slot_energies(d_stats, d_s2r, R, J, B, d_e, d_sums, sc));
    }
    PTMH_CUDA(cudaMemcpyAsync(h_small, d_small, n_out, cudaMemcpyDeviceToHost, sc));
    PTMH_CUDA(cudaStreamSynchronize(sc));
    PTMH_CUDA(cudaStreamSynchronize(sout));
    g_ws.dirty = false;
    memcpy(slot_to_row, h_small, 8 * R);
    memcpy(energies, h_small + o_e, 8 * R);
    memcpy(spin_sums, h_small + o_sums, 8 * R);
    int64_t cnt[2];
    memcpy(cnt, h_small + o_cnt, 16);
    if (accepted) *accepted = cnt[0];
    return PTMH_OK;
}
}  // extern "C"

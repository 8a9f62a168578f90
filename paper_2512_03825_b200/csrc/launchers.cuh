// launchers.cuh -- host-side launchers shared between the translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "philox.cuh"

namespace ptmh {

struct AdvanceArgs {
    int8_t* spins;
    int64_t L;
    const int64_t* slot_to_row;
    int64_t lo, hi;
    const double* tbl;   // (R, 10) exp(-beta_k * dE_c), host-built
    const double* dcls;  // (10) dE_c
    int int_energy;
    double* energies;
    int64_t* spin_sums;
    uint64_t* positions;
    int64_t* iters_done;
    uint64_t seed;
    int64_t start_iter, nsteps;
    double* obs_e;
    double* obs_m;
    int64_t ncols;
    int record;
    int8_t* states;
    uint32_t* bits;  // bit-packed lattices (row-major bits, ceil(L*L/32) words per row) or null
    uint64_t stream_offset;  // advance_kernel only: slot k draws from stream k + stream_offset
                             // (a lone replica's RngStream id, mh.py:73-88); 0 = the reference
};

// exact.cu (n = sites per lattice row)
int launch_fill(int8_t* spins, int64_t rows, int64_t n, int64_t up_count, uint64_t seed,
                uint64_t stream0, uint64_t pos0, cudaStream_t s);
int launch_row_stats(const int8_t* spins, int64_t rows, int64_t L, int64_t* stats, cudaStream_t s);
// init.cu (n = sites per lattice row)
int64_t fill_ws_bytes(int64_t n, int64_t rows_per_batch);
int launch_fill_parallel(int8_t* spins, int64_t rows, int64_t n, int64_t up_count, uint64_t seed,
                         uint64_t stream0, uint64_t pos0, void* ws, int64_t ws_bytes, cudaStream_t s);
int launch_advance(const AdvanceArgs& a, cudaStream_t s);
// swap rounds run inside the resident exact commit (exact.cu)
struct ExactRounds {
    int64_t swap_every;   // attempts per interval (0: no rounds)
    int64_t total_iters;  // N: rounds fire at completed = (k+1) * I < N
    const double* betas;  // by slot
    int64_t* counters;    // accepted, near ties
};
int launch_advance_2phase(const AdvanceArgs& a, void* ws, int64_t ws_bytes, cudaStream_t s,
                          const ExactRounds* rounds = nullptr);
int64_t advance_ws_bytes(int64_t nslots, int64_t nsteps);
int launch_bits_pack(const int8_t* spins, int64_t rows, int64_t L, uint32_t* bits, cudaStream_t s);
int launch_bits_unpack(const uint32_t* bits, int64_t rows, int64_t L, int8_t* spins, cudaStream_t s);
// n consecutive uniforms of one stream (rng.py:64-67, RngStream.uniform)
int launch_uniforms(uint64_t seed, uint64_t stream, uint64_t pos0, int64_t n, double* out, cudaStream_t s);
// reference swap rule for an explicit pair list (tempering.py:68-86): pair k
// draws from stream stream_base + k at position round_index; accept[k] = 0/1
int launch_swap_pairs(const int64_t* pi, const int64_t* pj, int64_t npairs, const double* betas,
                      const double* energies, uint64_t seed, int64_t stream_base, int64_t round_index,
                      uint8_t* accept, int64_t* near_ties, cudaStream_t s);
// the resident rounds' pair decision (rounds.cuh swap_decide) over given inputs
int launch_swap_decide(const double* bd, const double* Ei, const double* Ej, const double* u, int64_t n,
                       uint8_t* accept, uint8_t* near, cudaStream_t s);
int launch_swap(int64_t* slot_to_row, double* energies, int64_t* spin_sums, const double* betas,
                int64_t R, uint64_t seed, int64_t stream_base, int64_t round_index, int64_t first,
                int64_t pair_lo, int64_t pair_hi, int64_t* accepted, int64_t* near_ties,
                int32_t* row_to_slot, cudaStream_t s, const int64_t* stats = nullptr, double J = 0.0,
                double B = 0.0);

// checkerboard.cu
int64_t cb_words(int64_t L);
int launch_cb_sweeps(uint32_t* packed, int64_t rows, int64_t L, const int32_t* row_to_slot,
                     const uint32_t* thresh, uint32_t always_mask, uint64_t seed, int64_t first_sweep,
                     int64_t n_sweeps, int64_t* stats, cudaStream_t s, uint32_t* sync = nullptr,
                     uint32_t* scratch = nullptr);
// kind: 0 none, 1 cb_sweeps_persistent<rows, threads>, 2 cb_half_sweep_ferro<rows>,
// 3 cb_half_sweep_fast, 4 cb_half_sweep_generic; resident runs (resident.cu):
// 5 cb_resident_kernel (grid-barrier rounds; rows = cluster size),
// 6 cb_resident_p2p_kernel (warp-owned lattices), 7 cb_resident_kernel on
// clusters with point-to-point rounds, 8 cb_cluster_smem_kernel (rows = strip
// rows, group = cluster size; resident_smem.cu), 9 cb_resident_reg64_kernel
// (64^2 lattices in registers; resident_reg.cu), 10 cb_resident_reg32_kernel
// (32^2 lattices in registers)
struct CbLaunchInfo {
    int kind, rows, threads, group, bands, grid;
};
CbLaunchInfo cb_last_launch();
void cb_set_last_launch(const CbLaunchInfo& info);
bool cb_sweeps_persistent_applies(int64_t L, uint32_t always_mask, int64_t n_sweeps);
int launch_cb_pack(const int8_t* spins, int64_t rows, int64_t L, uint32_t* packed, cudaStream_t s);
int launch_cb_unpack(const uint32_t* packed, int64_t rows, int64_t L, int8_t* spins, cudaStream_t s);
int launch_cb_row_stats(const uint32_t* packed, int64_t rows, int64_t L, int64_t* stats, cudaStream_t s);
int launch_cb_unpack_slots(const uint32_t* packed, const int64_t* s2r, int64_t R, int64_t L, int8_t* out,
                           cudaStream_t s);
int launch_cb_slot_energies(const int64_t* stats, const int64_t* s2r, int64_t R, double J, double B,
                            double* energies, int64_t* sums, cudaStream_t s);
int launch_cb_observe(const int64_t* stats, const int64_t* s2r, int64_t R, int64_t L, double J, double B,
                      double* obs_e, double* obs_m, int64_t ncols, int64_t col, cudaStream_t s);

// resident.cu: one cooperative launch = many sweeps + exchange rounds
struct ResidentArgs {
    uint32_t* packed;  // (R, 2, W)
    int R, L, W, WR;   // WR = L/64 when L % 64 == 0, else 0 (generic gather)
    const uint32_t* thresh;
    RoundKeys32 rk;
    uint64_t seed;
    double J, B;
    const double* betas;
    int64_t* s2r[2];   // double-buffered slot_to_row
    int32_t* r2s[2];   // double-buffered row_to_slot
    int64_t* stats;    // (R, 2)
    int64_t* slot_stats;  // (2, R, 2): (S, Bond) by slot, buffer = round parity
    int64_t* counters; // accepted, near ties
    double* obs_e;
    double* obs_m;
    int64_t ncols;
    int64_t first_sweep, n_sweeps, total_sweeps;
    int64_t swap_every;    // sweeps, 0 = never
    int64_t record_every;  // 0 = no recording
    int buf;               // permutation buffer holding the current mapping
    int n_up, up_k[10], up_sf[10], up_cls[10];
    int ferro;
    uint32_t seg_lo, seg_even;  // L in {8, 16, 32}: bit 0 of each row segment, even-row segments
    int warp_lat;               // launcher-set: each warp owns whole lattices (no CTA barrier per colour)
    int strip;                  // launcher-set: warp-owned 64^2 ferro lattices use the strip code
    int p2p;                    // launcher-set: cluster-owned lattices decide rounds pairwise (u_table)
    int local_ring;             // launcher-set: one CTA holds every lattice, round words in shared memory
    // Sharded across GPUs (world > 1): R above counts this rank's lattices
    // (global rows row_lo ..), slots and pairs range over R_total.  Each
    // round's (S, Bond) by slot goes to every rank's pub buffer (peer memory
    // over NVLink), then one flag per (source rank) in every rank's flags
    // array; a rank proceeds when all flags reached round + 1.
    int world, rank, R_total;
    int64_t row_lo;
    int64_t* pub_peer[8];    // slot_stats (2, R_total, 2) of every rank (peer pointers), [rank] = own
    uint32_t* flag_peer[8];  // flags (world) of every rank, [rank] = own
    int max_ctas;            // 0 = fill the GPU (tests cap it to co-run virtual ranks on one GPU)
    // Point-to-point rounds (cb_resident_p2p_kernel): the swap draws of this
    // segment's rounds, u_table[(round - u_round0) * u_stride + pair]
    // (filled by swap_draws_kernel before the launch); null = grid-barrier rounds
    const double* u_table;
    int64_t u_round0, u_stride;
};
int launch_cb_resident(const ResidentArgs& a, bool fast, cudaStream_t s, int* grid_out);
// resident_smem.cu: ferro lattices held in the shared memory of a cluster of
// CTAs each (point-to-point rounds); returns 1 when it does not apply
int launch_cb_cluster_smem(const ResidentArgs& a, cudaStream_t s);
// resident_reg.cu: 64^2 ferro lattices held in registers, one warp each
// (grid CTAs of `threads`); returns 1 when it does not apply
int launch_cb_resident_reg64(const ResidentArgs& a, int grid, int threads, cudaStream_t s);
int launch_cb_resident_reg32(const ResidentArgs& a, int grid, int threads, cudaStream_t s);
// workspace of the point-to-point rounds: the swap draws of n_rounds rounds
int64_t resident_ws_bytes(int64_t R, int64_t n_rounds);
void fill_class_plan(uint32_t always_mask, int* n_up, int* k, int* sf, int* cls, int* ferro);

}  // namespace ptmh

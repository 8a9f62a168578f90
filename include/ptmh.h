/*
 * ptmh.h -- C ABI of the B200 Parallel-Tempering Metropolis engine.
 *
 * Plain C types only.  Two groups of entry points:
 *
 *  (A) Host-buffer entry points, ptmh_host_*: exactly the reference's kernel
 *      boundary.  The reference executor calls the numba kernels in
 *      isingpt/kernels.py as module attributes (executor.py:23,204-206,
 *      218-220,241-245,258-260) on caller-owned, C-contiguous host arrays
 *      that the kernels mutate in place.  Each ptmh_host_* function takes
 *      the same arrays (host pointers + shapes), copies them to the device,
 *      runs the CUDA kernel and copies the results back, so a ctypes binding
 *      can be installed as isingpt.kernels.<name>.
 *
 *  (B) Device-resident entry points: the same operations on device pointers
 *      (torch-allocated), asynchronous on the given cudaStream_t, plus the
 *      checkerboard (Mode F) sweep, pack/unpack and observable kernels.  The
 *      engine (paper_2512_03825_b200/engine.py) keeps every replica's state
 *      in HBM for the whole run and only calls these.
 *
 * Conventions: every function returns 0 (PTMH_OK) or a negative code;
 * ptmh_last_error() returns the message of the calling thread's last error.
 * No device function allocates or synchronises except the ptmh_host_* ones.
 */
#ifndef PTMH_H_
#define PTMH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PTMH_OK 0
#define PTMH_ERR_ARG (-1)
#define PTMH_ERR_CUDA (-2)

#define PTMH_ABI_VERSION 1

int ptmh_abi_version(void);
const char *ptmh_last_error(void);

/* ------------------------------------------------ (A) host-buffer ABI -- */

/* isingpt/kernels.py:26-27 fill_lattice(out, up_count, seed, stream, position)
 * -> new position.  out: int8 host array of n sites (any 2D shape). */
int ptmh_host_fill_lattice(int8_t *out, int64_t n, int64_t up_count,
                           uint64_t seed, uint64_t stream, uint64_t position,
                           uint64_t *new_position);

/* isingpt/kernels.py:48-49 lattice_energy(spins, J, B) -> float.
 * spins: int8 host (L, L). */
int ptmh_host_lattice_energy(const int8_t *spins, int64_t L, double J, double B,
                             double *energy);

/* isingpt/kernels.py:62-65 advance_block(spins, slot_to_row, lo, hi, betas, J,
 * B, energies, spin_sums, positions, iters_done, seed, start_iter, nsteps,
 * obs_e, obs_m, record, states).
 *   spins (rows, L, L) int8; slot_to_row/betas/energies/spin_sums/positions/
 *   iters_done: R entries; obs_e/obs_m (R, ncols) f64 (ignored if record==0);
 *   states (R, ncols, L, L) int8 (only if record==2). */
int ptmh_host_advance_block(int8_t *spins, int64_t rows, int64_t L,
                            const int64_t *slot_to_row, int64_t R, int64_t lo,
                            int64_t hi, const double *betas, double J, double B,
                            double *energies, int64_t *spin_sums,
                            uint64_t *positions, int64_t *iters_done,
                            uint64_t seed, int64_t start_iter, int64_t nsteps,
                            double *obs_e, double *obs_m, int64_t ncols,
                            int record, int8_t *states);

/* isingpt/kernels.py:116-118 swap_chunk(slot_to_row, energies, spin_sums,
 * betas, seed, stream_base, round_index, first, pair_lo, pair_hi) -> int. */
int ptmh_host_swap_chunk(int64_t *slot_to_row, double *energies,
                         int64_t *spin_sums, const double *betas, int64_t R,
                         uint64_t seed, int64_t stream_base,
                         int64_t round_index, int64_t first, int64_t pair_lo,
                         int64_t pair_hi, int64_t *accepted);

/* The reference's per-replica public ops on the device (host buffers).
 *
 * rng.py:64-96 RngStream.uniform / stream_uniform: out[t] = the uniform
 * (w >> 11) * 2^-53 of Philox4x64-10 word 0 at (seed, stream, position + t),
 * t = 0 .. n-1.  An RngStream then advances its position by n. */
int ptmh_host_uniforms(uint64_t seed, uint64_t stream, uint64_t position,
                       int64_t n, double *out);

/* tempering.py:68-86 execute_swap_round, decisions only: pair k = (pair_i[k],
 * pair_j[k]) indexes betas / energies (n entries) and draws
 * SwapRng.pair_uniform(round_index, k) = stream stream_base + k at position
 * round_index (rng.py:113-116); accept[k] = (u < swap_probability).  The
 * caller swaps its replicas' lattices and energies.  near_ties: decisions a
 * last-ulp exp difference could flip (expected 0). */
/* The resident kernels' exchange decision (kernels.py:116-148 rule, with an
 * FP32 fast path and the exact FP64 evaluation within 1e-5 of the boundary)
 * over n given (beta_i - beta_j, E_i, E_j, u) on the device: accept[t] = 1 iff
 * u < p; near[t] = 1 where |u - p| <= 4 ulp (a last-ulp exp difference from
 * glibc could flip it).  Device pointers; for tests of the decision. */
int ptmh_swap_decide(const double *bd, const double *Ei, const double *Ej,
                     const double *u, int64_t n, uint8_t *accept, uint8_t *near,
                     void *stream);

int ptmh_host_swap_pairs(const int64_t *pair_i, const int64_t *pair_j,
                         int64_t npairs, const double *betas,
                         const double *energies, int64_t n, uint64_t seed,
                         int64_t stream_base, int64_t round_index,
                         uint8_t *accept, int64_t *near_ties);

/* mh.py:73-88 mh_step, nsteps times, on one replica: lattice (L, L) int8,
 * cached energy and spin sum, RngStream (seed, stream, *position).  Each step
 * consumes two draws (site, acceptance), exactly as advance_block does for a
 * slot whose stream id is `stream` (kernels.py:62-113). */
int ptmh_host_mh_steps(int8_t *spins, int64_t L, double beta, double J,
                       double B, double *energy, int64_t *spin_sum,
                       uint64_t seed, uint64_t stream, uint64_t *position,
                       int64_t nsteps);

/* Checkerboard interval on host lattices (Mode F): the
 * plugin call bench.py times end to end.  Copies the int8 lattices
 * (rows, L, L) in, runs n_sweeps checkerboard sweeps starting at global
 * sweep first_sweep and -- if round_index >= 0 -- one swap round with the
 * reference rule, and copies the lattices, slot_to_row (R), by-slot
 * energies / spin sums (R) back.  Copies are pipelined over replica chunks
 * against the sweeps.  rows == R (single device). */
int ptmh_host_cb_interval(int8_t *spins, int64_t R, int64_t L,
                          int64_t *slot_to_row, const double *betas, double J,
                          double B, uint64_t seed, int64_t first_sweep,
                          int64_t n_sweeps, int64_t round_index,
                          double *energies, int64_t *spin_sums,
                          int64_t *accepted);

/* ---------------------------------------- (B) device-resident ABI ------ */

/* fill_lattice for rows [0, rows): row r uses stream stream0 + r from
 * position pos0 (executor.py:203-205).  spins: device (rows, L, L) int8. */
int ptmh_fill_lattices(int8_t *spins, int64_t rows, int64_t L,
                       int64_t up_count, uint64_t seed, uint64_t stream0,
                       uint64_t pos0, void *stream);

/* The same lattices as ptmh_fill_lattices, bit for bit, computed in parallel
 * (csrc/init.cu: every draw at once, the swaps resolved through per-position
 * writer lists).  workspace: ptmh_fill_workspace_bytes(L, k) bytes processes
 * k rows per pass. */
int64_t ptmh_fill_workspace_bytes(int64_t L, int64_t rows_per_batch);
int ptmh_fill_lattices_parallel(int8_t *spins, int64_t rows, int64_t L,
                                int64_t up_count, uint64_t seed, uint64_t stream0,
                                uint64_t pos0, void *workspace, int64_t ws_bytes,
                                void *stream);

/* The sweep kernel the calling thread's last ptmh_cb_sweeps / _sync call
 * launched: info[0] = kind (0 none, 1 cb_sweeps_persistent<rows, threads>,
 * 2 cb_half_sweep_ferro<rows>, 3 cb_half_sweep_fast, 4 cb_half_sweep_generic;
 * info[4] = 2: temporally blocked items (ptmh_cb_sweeps_ws), 3: the same
 * streamed through each band (states of more than 2^25 sites);
 * after a resident run: 5 cb_resident_kernel with grid-barrier rounds, 6
 * cb_resident_p2p_kernel, 7 cb_resident_kernel on clusters with
 * point-to-point rounds; info[1] = cluster size there; 8
 * cb_cluster_smem_kernel, lattices in the shared memory of clusters of
 * info[3] CTAs, info[1] = strip rows; 9 cb_resident_reg64_kernel, 64^2
 * lattices held in registers, a warp each; 10 cb_resident_reg32_kernel,
 * the same for 32^2),
 * info[1] = rows per thread, [2] = threads per item / CTA, [3] = blocks per
 * item (group), [4] = band dependencies, [5] = grid (persistent only). */
int ptmh_cb_last_launch(int32_t *info);

/* rng.py:64-67 stream_uniform for positions position .. position+n-1 of one
 * stream, into device memory. */
int ptmh_uniforms(uint64_t seed, uint64_t stream_id, uint64_t position,
                  int64_t n, double *out, void *stream);

/* stats[2r] = sum(s), stats[2r+1] = sum(s*(down+right)) of each int8 lattice
 * (the integer accumulators of kernels.py:48-59). */
int ptmh_row_stats(const int8_t *spins, int64_t rows, int64_t L,
                   int64_t *stats, void *stream);

/* advance_block on device arrays.  The acceptance exponentials are built on
 * the host with the reference's own expression and libm exp:
 *   dcls[c]      = 2.0*s*(J*nb - B),  c = 5*(s>0) + (nb+4)/2   (10 classes)
 *   tbl[k*10+c]  = exp(-betas[k]*dcls[c])                      (R x 10)
 * int_energy != 0 allows order-free energy accumulation (integer J, B). */
int ptmh_advance_block(int8_t *spins, int64_t L, const int64_t *slot_to_row,
                       int64_t lo, int64_t hi, const double *tbl,
                       const double *dcls, int int_energy, double *energies,
                       int64_t *spin_sums, uint64_t *positions,
                       int64_t *iters_done, uint64_t seed, int64_t start_iter,
                       int64_t nsteps, double *obs_e, double *obs_m,
                       int64_t ncols, int record, int8_t *states, void *stream);

/* Two-phase advance_block (record 0 or 1; obs_e == NULL means record 0):
 * phase 1 computes every attempt's draws, site, per-class acceptance bits and
 * window dependencies fully in parallel into `workspace`
 * (ptmh_advance_workspace_bytes(hi-lo, nsteps) bytes); phase 2 commits them
 * warp-per-slot.  Results identical to ptmh_advance_block. */
int64_t ptmh_advance_workspace_bytes(int64_t nslots, int64_t nsteps);
int ptmh_advance_block_ws(int8_t *spins, int64_t L, const int64_t *slot_to_row,
                          int64_t lo, int64_t hi, const double *tbl,
                          const double *dcls, int int_energy, double *energies,
                          int64_t *spin_sums, uint64_t *positions,
                          int64_t *iters_done, uint64_t seed, int64_t start_iter,
                          int64_t nsteps, double *obs_e, double *obs_m,
                          int64_t ncols, void *workspace, int64_t ws_bytes,
                          void *stream);

/* Bit-packed exact-chain lattices: site x of row r is bit (x & 31) of word
 * bits[r*ceil(L*L/32) + (x >> 5)], set <=> +1.  ptmh_advance_block_bits is
 * ptmh_advance_block_ws on that representation (same results; 1 bit per spin
 * keeps large lattice sets L2-resident for the random-site commits). */
int ptmh_bits_pack(const int8_t *spins, int64_t rows, int64_t L, uint32_t *bits,
                   void *stream);
int ptmh_bits_unpack(const uint32_t *bits, int64_t rows, int64_t L,
                     int8_t *spins, void *stream);
int ptmh_advance_block_bits(uint32_t *bits, int64_t L, const int64_t *slot_to_row,
                            int64_t lo, int64_t hi, const double *tbl,
                            const double *dcls, int int_energy,
                            double *energies, int64_t *spin_sums,
                            uint64_t *positions, int64_t *iters_done,
                            uint64_t seed, int64_t start_iter, int64_t nsteps,
                            double *obs_e, double *obs_m, int64_t ncols,
                            void *workspace, int64_t ws_bytes, void *stream);

/* swap_chunk on device arrays; accepted[0] += accepted pairs, near_ties[0] +=
 * decisions with |u - p| <= 4 ulp(p) (device exp vs host libm guard band).
 * If row_to_slot is non-NULL it is rebuilt from slot_to_row afterwards. */
int ptmh_swap_chunk(int64_t *slot_to_row, double *energies, int64_t *spin_sums,
                    const double *betas, int64_t R, uint64_t seed,
                    int64_t stream_base, int64_t round_index, int64_t first,
                    int64_t pair_lo, int64_t pair_hi, int64_t *accepted,
                    int64_t *near_ties, int32_t *row_to_slot, void *stream);

/* One checkerboard exchange round in one launch: energies[k] / spin_sums[k]
 * of slot k from the per-lattice stats (as ptmh_cb_slot_energies), then the
 * reference swap rule for round_index (as ptmh_swap_chunk with stream_base R,
 * all pairs), then row_to_slot rebuilt. */
int ptmh_cb_exchange(const int64_t *stats_all, int64_t *slot_to_row,
                     int32_t *row_to_slot, int64_t R, double J, double B,
                     const double *betas, uint64_t seed, int64_t round_index,
                     double *energies, int64_t *spin_sums, int64_t *accepted,
                     int64_t *near_ties, void *stream);

/* Checkerboard (Mode F) storage: per lattice, colour c in {0,1}, half-lattice
 * site h = i*(L/2) + (j>>1) of colour (i+j)&1 is bit (h & 31) of word
 * packed[(row*2 + c)*W + (h >> 5)], W = ceil(L*L/64); bit set <=> spin +1. */
int64_t ptmh_cb_words_per_color(int64_t L);
int ptmh_cb_pack(const int8_t *spins, int64_t rows, int64_t L, uint32_t *packed,
                 void *stream);
int ptmh_cb_unpack(const uint32_t *packed, int64_t rows, int64_t L,
                   int8_t *spins, void *stream);

/* out (R, L, L) int8: lattice slot_to_row[k] unpacked into out[k] (by slot;
 * full_states recording). */
int ptmh_cb_unpack_slots(const uint32_t *packed, const int64_t *slot_to_row,
                         int64_t R, int64_t L, int8_t *out, void *stream);

/* n_sweeps checkerboard sweeps (colour 0 then 1) of rows [0, rows) starting
 * at global sweep first_sweep.  Row r is at slot row_to_slot[r] (global slot
 * index; row_offset is the global index of local row 0, unused by the
 * kernel but kept for sharded callers).  thresh: (R, 10) uint32, always_mask:
 * the classes with dE <= 0.  stats (rows, 2) int64 is updated incrementally
 * (fused reduction). */
int ptmh_cb_sweeps(uint32_t *packed, int64_t rows, int64_t L,
                   const int32_t *row_to_slot, const uint32_t *thresh,
                   uint32_t always_mask, uint64_t seed, int64_t first_sweep,
                   int64_t n_sweeps, int64_t *stats, void *stream);

/* ptmh_cb_sweeps with a caller-owned sync block (uint32, ptmh_cb_sync_words
 * (rows, L) words, zeroed once; every call leaves it zeroed).  With it, the
 * J > 0, B = 0, L % 512 == 0, L >= 1024 case runs all 2 * n_sweeps half-sweeps in ONE
 * persistent launch (a dataflow over work items with per-band dependencies,
 * no grid-wide barrier between colours); other cases, or sync == NULL, take
 * the per-launch path.  Results are bit-identical either way.  Calls sharing
 * a sync block must be ordered on one stream. */
int64_t ptmh_cb_sync_words(int64_t rows, int64_t L);
int ptmh_cb_sweeps_sync(uint32_t *packed, int64_t rows, int64_t L,
                        const int32_t *row_to_slot, const uint32_t *thresh,
                        uint32_t always_mask, uint64_t seed,
                        int64_t first_sweep, int64_t n_sweeps, int64_t *stats,
                        uint32_t *sync, void *stream);

/* ptmh_cb_sweeps_sync with a caller-owned scratch state buffer of the
 * packed state's size (rows * 2 * ceil(L*L/64) uint32, contents irrelevant):
 * the persistent path then runs temporally blocked -- one work item per
 * (sweep, lattice, band), both colours of the band, out of place between
 * packed and scratch (ping-pong), so every word is read once per sweep
 * instead of once per colour.  The result is in `packed` afterwards (an odd
 * sweep count ends with one device copy).  stats (rows, 2) are overwritten
 * with the final (S, Bond), as on every other path.  Bit-identical to
 * ptmh_cb_sweeps.  scratch == NULL is ptmh_cb_sweeps_sync. */
int ptmh_cb_sweeps_ws(uint32_t *packed, int64_t rows, int64_t L,
                      const int32_t *row_to_slot, const uint32_t *thresh,
                      uint32_t always_mask, uint64_t seed, int64_t first_sweep,
                      int64_t n_sweeps, int64_t *stats, uint32_t *sync,
                      uint32_t *scratch, void *stream);

/* Persistent single-device run segment (csrc/resident.cu): sweeps
 * first_sweep .. first_sweep+n_sweeps-1 of a run of total_sweeps sweeps,
 * with the swap rounds (every swap_every sweeps, strictly before the end,
 * executor.py:111-125) and observations (every record_every sweeps, by slot,
 * before the round; record_every 0 = none) inside ONE cooperative launch.
 * slot_to_row2 (2, R) int64 / row_to_slot2 (2, R) int32 are double buffers;
 * `buf` names the one holding the current permutation, *buf_out receives the
 * one holding it afterwards.  stats (R, 2) hold every lattice's (S, Bond)
 * after the segment.  slot_stats is caller-owned scratch of 4 * R int64 (the
 * per-slot (S, Bond) table an exchange round reads, double-buffered by round
 * parity).  Same chain and random numbers as ptmh_cb_sweeps. */
int ptmh_cb_run_resident(uint32_t *packed, int64_t R, int64_t L,
                         int64_t *slot_to_row2, int32_t *row_to_slot2, int buf,
                         const uint32_t *thresh, uint32_t always_mask,
                         uint64_t seed, double J, double B, const double *betas,
                         int64_t *stats, int64_t *slot_stats,
                         int64_t *counters, double *obs_e, double *obs_m,
                         int64_t ncols, int64_t first_sweep, int64_t n_sweeps,
                         int64_t total_sweeps, int64_t swap_every,
                         int64_t record_every, int *buf_out, void *stream);

/* ptmh_cb_run_resident with a workspace of ptmh_cb_resident_ws_bytes(R,
 * n_rounds) bytes (n_rounds: the segment's exchange rounds).  Where every
 * lattice has its own warp (small lattices, e.g. C5's 64^2 x 4096, C1), the
 * rounds are then decided pair by pair -- each lattice publishes its
 * (S, Bond) for its slot and waits only for its partner slot's -- instead of
 * behind a grid barrier (csrc/resident.cu, cb_resident_p2p_kernel); the
 * workspace holds the segment's swap draws.  Same chain, same results. */
int64_t ptmh_cb_resident_ws_bytes(int64_t R, int64_t n_rounds);
int ptmh_cb_run_resident_ws(uint32_t *packed, int64_t R, int64_t L,
                            int64_t *slot_to_row2, int32_t *row_to_slot2,
                            int buf, const uint32_t *thresh,
                            uint32_t always_mask, uint64_t seed, double J,
                            double B, const double *betas, int64_t *stats,
                            int64_t *slot_stats, int64_t *counters,
                            double *obs_e, double *obs_m, int64_t ncols,
                            int64_t first_sweep, int64_t n_sweeps,
                            int64_t total_sweeps, int64_t swap_every,
                            int64_t record_every, int *buf_out, void *ws,
                            int64_t ws_bytes, void *stream);

/* ptmh_cb_run_resident_sharded with the point-to-point rounds' workspace
 * (ptmh_cb_resident_ws_bytes(R_total, n_rounds)): where lattices are
 * warp-owned, every lattice stores its round word into every rank's
 * slot_stats ring (NVLink peer stores) and waits for its partner slot's word
 * only; flag_peers are then unused.  The rings must start zeroed for a run
 * (ptmh_peer_alloc) and a run's rounds only grow. */
int ptmh_cb_run_resident_sharded_ws(uint32_t *packed, int64_t rows, int64_t L,
                                    int64_t *slot_to_row2, int32_t *row_to_slot2,
                                    int buf, const uint32_t *thresh,
                                    uint32_t always_mask, uint64_t seed, double J,
                                    double B, const double *betas, int64_t *stats,
                                    int64_t *slot_stats, int64_t *counters,
                                    double *obs_e, double *obs_m, int64_t ncols,
                                    int64_t first_sweep, int64_t n_sweeps,
                                    int64_t total_sweeps, int64_t swap_every,
                                    int64_t record_every, int *buf_out,
                                    int64_t R_total, int rank, int world,
                                    int64_t row_lo, int64_t *const *pub_peers,
                                    uint32_t *const *flag_peers, int max_ctas,
                                    void *ws, int64_t ws_bytes, void *stream);

/* ptmh_cb_run_resident over `world` GPUs (one process each): this rank owns
 * the `rows` lattices of global rows row_lo .. row_lo + rows - 1; slots,
 * betas, thresholds, observables and slot_to_row2 (2, R_total) range over
 * R_total.  Each round's (S, Bond) by slot is stored into every rank's
 * slot_stats (pub_peers[g], peer pointers from ptmh_ipc_open; [rank] =
 * slot_stats) and signalled through flag_peers[g][rank] (uint32, world
 * entries per rank, zeroed once per run); no collective library call.  On
 * return this rank's row_to_slot2 / stats are current; counters, the
 * observables and slot_to_row2 hold only this rank's part (the caller
 * combines them).  max_ctas caps the grid (0: fill the GPU). */
int ptmh_cb_run_resident_sharded(uint32_t *packed, int64_t rows, int64_t L,
                                 int64_t *slot_to_row2, int32_t *row_to_slot2,
                                 int buf, const uint32_t *thresh,
                                 uint32_t always_mask, uint64_t seed, double J,
                                 double B, const double *betas, int64_t *stats,
                                 int64_t *slot_stats, int64_t *counters,
                                 double *obs_e, double *obs_m, int64_t ncols,
                                 int64_t first_sweep, int64_t n_sweeps,
                                 int64_t total_sweeps, int64_t swap_every,
                                 int64_t record_every, int *buf_out,
                                 int64_t R_total, int rank, int world,
                                 int64_t row_lo, int64_t *const *pub_peers,
                                 uint32_t *const *flag_peers, int max_ctas,
                                 void *stream);

/* CUDA IPC for the peer buffers above: handle_out receives
 * ptmh_ipc_handle_bytes() bytes. */
int64_t ptmh_ipc_handle_bytes(void);
int ptmh_ipc_handle(void *dev_ptr, void *handle_out);
int ptmh_ipc_open(const void *handle, void **dev_ptr_out);
int ptmh_ipc_close(void *dev_ptr);
/* zeroed cudaMalloc allocation for IPC-shared buffers (a handle names a whole
 * allocation, not a sub-block of a caching allocator's segment) */
int ptmh_peer_alloc(int64_t bytes, void **dev_ptr_out);
int ptmh_peer_free(void *dev_ptr);

/* The exact chain for iterations start_iter .. start_iter+nsteps-1 of a run
 * of total_iters, WITH its swap rounds (every swap_every iterations,
 * executor.py:111-125): draws on the whole GPU, then one CTA per chunk
 * commits every slot (R <= 32, bit lattices in shared memory) and runs the
 * rounds in between (csrc/exact.cu, exact_resident_kernel).  A call runs
 * the rounds at completed = start_iter .. start_iter+nsteps-1 (the one at its
 * first iteration before any attempt; the one at its end belongs to the next
 * call), so consecutive calls cover every round once.  slot_to_row,
 * energies, spin_sums are updated in place; counters += (accepted, near
 * ties).  Workspace: ptmh_advance_workspace_bytes(R, nsteps).  Bit-exact with
 * the reference's executor loop. */
int ptmh_exact_run_resident(uint32_t *bits, int64_t L, int64_t *slot_to_row,
                            int64_t R, const double *tbl, const double *dcls,
                            int int_energy, double *energies, int64_t *spin_sums,
                            uint64_t *positions, int64_t *iters_done,
                            uint64_t seed, int64_t start_iter, int64_t nsteps,
                            int64_t swap_every, int64_t total_iters,
                            const double *betas, int64_t *counters,
                            double *obs_e, double *obs_m, int64_t ncols,
                            void *workspace, int64_t ws_bytes, void *stream);

/* Per-lattice (S, Bond) recomputed from the packed state (audit of the
 * incremental stats; L % 64 == 0 or any even L). */
int ptmh_cb_row_stats(const uint32_t *packed, int64_t rows, int64_t L,
                      int64_t *stats, void *stream);

/* energies[k] = B*S - J*Bond and spin_sums[k] = S of lattice slot_to_row[k]
 * (lattice.py:61-65), for k in [0, R).  stats_all holds every lattice. */
int ptmh_cb_slot_energies(const int64_t *stats_all, const int64_t *slot_to_row,
                          int64_t R, double J, double B, double *energies,
                          int64_t *spin_sums, void *stream);

/* obs_e[k*ncols + col] = energy of slot k, obs_m[...] = S / L^2. */
int ptmh_cb_observe(const int64_t *stats_all, const int64_t *slot_to_row,
                    int64_t R, int64_t L, double J, double B, double *obs_e,
                    double *obs_m, int64_t ncols, int64_t col, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* PTMH_H_ */

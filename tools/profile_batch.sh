#!/bin/bash
# One gpurun batch behind the committed profiles (then: python tools/refresh_profiles.py r2):
#   bench lines for every config, the reference arm, the C3 launch list, ncu --set full captures of
#   the hot kernels, and the compute-sanitizer pass.
mkdir -p gpurun_out
for c in c3 c1 c2 c5; do python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; done
python bench.py --config c4 --steps 20 > gpurun_out/bench_c4.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --no-exact > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cb_sweeps_persistent -c 1 \
    -o gpurun_out/persist_c3 -f python tools/prof_sweep.py c3 10 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:cb_sweeps_persistent -c 1 \
    -o gpurun_out/persist_c4 -f python tools/prof_sweep.py c4 2 > /dev/null 2>&1
# C4 with temporally blocked items forced on (streamed through each band): DRAM bytes vs the default
PTMH_PERSIST_TB=1 ncu --set full --clock-control none -k regex:cb_sweeps_persistent -c 1 \
    -o gpurun_out/persist_c4_tbs -f python tools/prof_sweep.py c4 2 > /dev/null 2>&1
# a rank's C3 shard at 8 GPUs: the temporally blocked persistent launch
ncu --set full --clock-control none --import-source on -k regex:cb_sweeps_persistent -c 1 \
    -o gpurun_out/persist_shard32 -f python tools/prof_sweep.py 1024,32 10 > /dev/null 2>&1
tail -n 1 gpurun_out/bench_*.log
# the resident kernels, 20 sweeps with a round every sweep: C5 (warp-owned lattices) and C2
# (lattices in cluster shared memory; ncu replays the cooperative cluster launch only without the
# cooperative attribute, PTMH_SMEM_NOCOOP=1 -- every cluster is resident on an idle GPU either way)
ncu --set full --clock-control none --import-source on -k regex:cb_resident_reg64 -c 1 -o gpurun_out/res_c5 -f \
    python tools/prof_resident.py c5 1 > /dev/null 2>&1
PTMH_SMEM_NOCOOP=1 ncu --set full --clock-control none --import-source on -k regex:cb_cluster_smem -c 1 \
    -o gpurun_out/res_c2 -f python tools/prof_resident.py c2 1 > /dev/null 2>&1
# (compute-sanitizer: closed on the GPU pool since the last round-2 refresh; profiles/r2_sanitizer.txt
# holds the last pass, commit 03ae124: the kernels are unchanged since)

#!/bin/bash
# One gpurun batch behind the committed profiles (then: python tools/refresh_profiles.py r2):
#   bench lines for every config, the reference arm, the C3 launch list and an
#   ncu --set full capture of the C3 hot kernel.
mkdir -p gpurun_out
for c in c3 c1 c2 c5; do python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; done
python bench.py --config c4 --steps 20 > gpurun_out/bench_c4.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --no-exact > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cb_sweeps_persistent -c 1 \
    -o gpurun_out/persist_c3 -f python tools/prof_sweep.py c3 10 > gpurun_out/ncu_full.log 2>&1
tail -n 1 gpurun_out/bench_*.log
# the resident kernels (C5: warp-owned lattices, C2: clusters), 20 sweeps with a round every sweep
ncu --set full --clock-control none --import-source on -k regex:cb_resident -c 1 -o gpurun_out/res_c5 -f \
    python tools/prof_resident.py c5 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:cb_resident -c 1 -o gpurun_out/res_c2 -f \
    python tools/prof_resident.py c2 1 > /dev/null 2>&1

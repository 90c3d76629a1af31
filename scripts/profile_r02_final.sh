#!/bin/bash
# Final round-2 evidence: bench line, whole-step launch list, DMMA Galerkin captures.
set -u
O=gpurun_out/r02f
mkdir -p $O
python bench.py --steps 3 --warmup 3 > $O/bench.json 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file $O/launches_step.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > $O/launches_bench.log 2>&1
gzip -f $O/launches_step.csv
ncu --set full --clock-control none --kernel-name-base demangled -k regex:'k_galerkin' -s 0 -c 2 -o $O/galerkin \
    python scripts/profile_kernel.py c4_mbb_5120x2560 1 > $O/galerkin.log 2>&1
ncu --set full --clock-control none --kernel-name-base demangled -k regex:'k_galerkin_gemm' -s 0 -c 1 -o $O/galerkin_c3 \
    python scripts/profile_kernel.py c3_square_2048 1 > $O/galerkin_c3.log 2>&1
ls -la $O

#!/bin/bash
# Final round-2 evidence (one B200, through gpurun from the repo root): GPU tests, bench line,
# whole-step launch list, ncu --set full captures of the PCG's two sweeps (one and three
# realisations) and of the other PCG kernels.
set -u
O=gpurun_out/r02f2
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1
python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file $O/launches_step.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > $O/launches_bench.log 2>&1
gzip -f $O/launches_step.csv
cap() {   # name regex(demangled) skip count [nr]
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"$2" -s $3 -c $4 -o $O/$1 \
      python scripts/profile_kernel.py c4_mbb_5120x2560 ${5:-1} > $O/$1.log 2>&1
}
cap sgsw_pre 'k_sgs_warp<\(bool\)1, \(bool\)1' 3 1
cap sgsw_post 'k_sgs_warp<\(bool\)0, \(bool\)0, \(bool\)1' 3 1
cap sgsw_pre_3rhs 'k_sgs_warp<\(bool\)1, \(bool\)1' 3 1 3
cap sgsw_post_3rhs 'k_sgs_warp<\(bool\)0, \(bool\)0, \(bool\)1' 3 1 3
ls -la $O
tail -3 $O/gputests.log

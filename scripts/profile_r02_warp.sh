#!/bin/bash
# Round-2 evidence for the warp-synchronous sweep build (one B200, through gpurun from the repo
# root): bench line, whole-step launch list, ncu --set full captures of the two sweeps at one and
# three realisations and of the other PCG kernels.
set -u
O=gpurun_out/r02w
mkdir -p $O
python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file $O/launches_step.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > $O/launches_bench.log 2>&1
gzip -f $O/launches_step.csv
cap() {   # name regex(demangled) skip count [nr]
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"$2" -s $3 -c $4 -o $O/$1 \
      python scripts/profile_kernel.py c4_mbb_5120x2560 ${5:-1} > $O/$1.log 2>&1
}
cap sgsw_1rhs 'k_sgs_warp' 4 2
cap sgsw_3rhs 'k_sgs_warp' 4 2 3
cap pcg_rest 'k_apply_tma|k_restrict_cells|k_prolong_cells|k_pcg_p' 8 5
ls -la $O

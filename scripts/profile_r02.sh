#!/bin/bash
# Round-2 evidence on one B200 (run through gpurun from the repo root), in two parts so each
# call's gpurun_out stays under the 64 MiB copy-back limit:
#   bash scripts/profile_r02.sh A   whole-step launch list + the PCG kernels
#   bash scripts/profile_r02.sh B   coarse solve / factorisation / Galerkin / eigen / 3-realisation transfer
# Every capture: ncu --set full, configs[4], one realisation active unless noted.
set -u
O=gpurun_out/r02
mkdir -p $O
cap() {   # name regex(demangled) skip count [nr]
  ncu --set full --clock-control none --kernel-name-base demangled -k regex:"$2" -s $3 -c $4 -o $O/$1 \
      python scripts/profile_kernel.py c4_mbb_5120x2560 ${5:-1} > $O/$1.log 2>&1
}
if [ "${1:-A}" = A ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file $O/launches_step.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > $O/launches_bench.log 2>&1
  gzip -f $O/launches_step.csv
  cap sgs_pre 'k_sgs_warp<\(bool\)1, \(bool\)1' 0 1
  cap sgs_post 'k_sgs_warp<\(bool\)0, \(bool\)0, \(bool\)1' 1 1
  cap restrict 'k_restrict_cells' 1 1
  cap prolong 'k_prolong_cells' 1 1
else
  cap apply 'k_apply_tma<\(int\)0' 1 1
  cap residual 'k_apply_tma<\(int\)1' 1 1
  cap pcg_p 'k_pcg_p' 1 1
  cap nd_solve 'k_nd_solve' 0 6
  cap nd_factor 'k_nd_trailing|k_nd_panels|k_nd_rowpanel|k_nd_pivot|k_nd_assemble' 0 8
  cap galerkin 'k_cell_galerkin' 0 1
  cap eigen 'k_eigen' 0 2
  cap xfer_3rhs 'k_restrict_cells|k_prolong_cells' 2 2 3
fi
ls -la $O

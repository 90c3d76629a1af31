#!/bin/bash
# Round-2 evidence on one B200 (run through gpurun from the repo root): the whole-step launch
# list of the bench command and one `ncu --set full` capture per hot kernel (configs[4], one
# realisation active unless noted).  Reports land in gpurun_out/; summaries go to profiles/.
set -u
O=gpurun_out/r02
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file $O/launches_step.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > $O/launches_bench.log 2>&1
gzip -f $O/launches_step.csv
cap() {   # name regex skip count [nr]
  ncu --set full --import-source on --clock-control none -k regex:"$2" -s $3 -c $4 -o $O/$1 \
      python scripts/profile_kernel.py c4_mbb_5120x2560 ${5:-1} > $O/$1.log 2>&1
}
cap sgs_pre 'k_sgs_stream<1, 1' 0 1
cap sgs_post 'k_sgs_stream<0, 0, 0' 1 1
cap apply 'k_apply_tma<0' 1 1
cap residual 'k_apply_tma<1' 1 1
cap restrict 'k_restrict_cells' 1 1
cap prolong 'k_prolong_cells' 1 1
cap pcg_p 'k_pcg_p' 1 1
cap nd_solve 'k_nd_solve' 0 12
cap nd_factor 'k_nd_trailing|k_nd_panels|k_nd_rowpanel|k_nd_pivot|k_nd_assemble' 0 16
cap galerkin 'k_cell_galerkin' 0 1
cap eigen 'k_eigen' 0 3
cap xfer_3rhs 'k_restrict_cells|k_prolong_cells' 2 2 3
ls -la $O

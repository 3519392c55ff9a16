#!/bin/bash
# Round-2 session-5 profile batch (after the per-kernel shared-memory limits moved to allow_dyn_smem and the
# staged pageable upload): launch list of the default bench command, one full ncu capture of the dominant kernel.
set -u
O=gpurun_out
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $O/r02s5_launches_cfg2.csv \
  python bench.py --workload cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > $O/r02s5_ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rhqr_col_kernel -s 200 -c 1 -f -o $O/r02s5_col_cfg2 \
  python bench.py --workload cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > $O/r02s5_ncu_col2.log 2>&1; echo "cfg2 col rc=$?"
ls -la $O | grep r02s5

#!/bin/bash
# Round-2 measurement batch (run under gpurun from the repo root): tests, bench
# lines of every config, the launch list of the default bench command and full
# ncu captures of the dominant kernels.  Everything lands in gpurun_out/.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/r02f_pytest.log 2>&1; tail -2 $O/r02f_pytest.log
timeout 600 python bench.py > $O/r02f_bench_default.json 2> $O/r02f_bench_default.err; echo "bench default rc=$?"
: > $O/r02f_bench_all.jsonl
for w in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 2>> $O/r02f_bench_all.err | grep '^{' >> $O/r02f_bench_all.jsonl
done
wc -l $O/r02f_bench_all.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $O/r02f_launches_cfg2.csv \
  python bench.py --workload cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > $O/r02f_ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rhqr_col_kernel -s 200 -c 1 -f -o $O/r02f_col_cfg2 \
  python bench.py --workload cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > $O/r02f_ncu_col2.log 2>&1; echo "cfg2 col rc=$?"
PN=16777216 timeout 600 ncu --set full --clock-control none --import-source on -k regex:rhqr_col_kernel -s 127 -c 1 -f -o $O/r02f_col_cfg4 \
  python scripts/prof_cfg4.py > $O/r02f_ncu_col4.log 2>&1; echo "cfg4 col rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:rhqr_persist_fast -s 2 -c 1 -f -o $O/r02f_persist_cfg1 \
  python scripts/prof_cfg1.py > $O/r02f_ncu_persist.log 2>&1; echo "cfg1 persist rc=$?"
PROF_TAG=bf16 timeout 300 ncu --set full --clock-control none --import-source on -k regex:srht_tma16_tile -s 1 -c 1 -f -o $O/r02f_srht_bf16 \
  python scripts/prof_srht.py > $O/r02f_ncu_srht16.log 2>&1; echo "srht bf16 rc=$?"
for c in 4 2; do CFG=$c COLS=16,64,128 timeout 300 python scripts/col_timeline.py > $O/r02f_timeline_cfg$c.txt 2>&1; done
ls -la $O | tail -20

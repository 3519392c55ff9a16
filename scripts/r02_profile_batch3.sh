#!/bin/bash
# Round-2 final measurement batch: tests, smoke, bench lines of every config (ours + reference arm),
# launch list of the default bench command, full ncu captures of the dominant kernels.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/r02z_pytest.log 2>&1; tail -2 $O/r02z_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r02z_smoke.log 2>&1; tail -1 $O/r02z_smoke.log
timeout 900 python bench.py > $O/r02z_bench_default.json 2> $O/r02z_bench_default.err; echo "bench default rc=$?"
: > $O/r02z_bench_all.jsonl
for w in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 2>> $O/r02z_bench_all.err | grep '^{' >> $O/r02z_bench_all.jsonl
done
wc -l $O/r02z_bench_all.jsonl
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/r02z_bench_reference.json 2> $O/r02z_bench_reference.err; echo "reference arm rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $O/r02z_launches_cfg2.csv \
  python bench.py --workload cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > $O/r02z_ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rhqr_col_kernel -s 200 -c 1 -f -o $O/r02z_col_cfg2 \
  python bench.py --workload cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-other-configs > $O/r02z_ncu_col2.log 2>&1; echo "cfg2 col rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:rhqr_persist_fast -s 2 -c 1 -f -o $O/r02z_persist_cfg1 \
  python scripts/prof_cfg1.py > $O/r02z_ncu_persist.log 2>&1; echo "cfg1 persist rc=$?"
timeout 300 python scripts/persist_phases.py > $O/r02z_persist_phases.txt 2>&1
timeout 300 python scripts/trace_cfg5.py > $O/r02z_trace_cfg5.txt 2>&1
timeout 300 python scripts/trace_paths.py > $O/r02z_trace_paths.txt 2>&1
timeout 300 python scripts/trace_paths2.py > $O/r02z_trace_paths2.txt 2>&1
ls -la $O | grep r02z

#!/bin/bash
# Round-2 session-4 measurement batch after the K2 TMA kernel / DMMA diagnostics / fused exchange.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/r02g_pytest.log 2>&1; tail -2 $O/r02g_pytest.log
timeout 600 python bench.py > $O/r02g_bench_default.json 2> $O/r02g_bench_default.err; echo "bench default rc=$?"
: > $O/r02g_bench_all.jsonl
for w in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 2>> $O/r02g_bench_all.err | grep '^{' >> $O/r02g_bench_all.jsonl
done
wc -l $O/r02g_bench_all.jsonl
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/r02g_bench_reference.json 2> $O/r02g_bench_reference.err; echo "reference arm rc=$?"
REPS=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file $O/r02g_launches_cfg3.csv \
  python scripts/prof_cfg3.py > $O/r02g_ncu_launches3.log 2>&1; echo "cfg3 launch list rc=$?"
REPS=2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:dense_tma_kernel -s 1 -c 1 -f -o $O/r02g_dense_tma \
  python scripts/prof_cfg3.py > $O/r02g_ncu_dense.log 2>&1; echo "cfg3 dense rc=$?"
timeout 300 python scripts/dist_world1.py > $O/r02g_dist_world1.txt 2>&1
timeout 300 python scripts/trace_paths.py > $O/r02g_trace_paths.txt 2>&1
timeout 300 python scripts/trace_cfg5.py > $O/r02g_trace_cfg5.txt 2>&1
ls -la $O | tail -14

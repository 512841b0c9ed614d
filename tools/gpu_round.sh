#!/bin/bash
# One GPU call: tests, bench (both arms), ncu launch list + full captures.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${NCU_TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/host.txt; lscpu | head -20 >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
fi
if [ "${SKIP_BENCH:-0}" != "1" ]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -c 600 gpurun_out/bench.json
fi
if [ "${SKIP_REF:-0}" != "1" ]; then
  timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
  tail -c 400 gpurun_out/bench_ref.json
fi
if [ "${SKIP_NCU:-0}" != "1" ]; then
  CMD="python bench.py --steps 20 --warmup 3 --no-extra --no-cpu-baseline"
  $CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  CMD4="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu-baseline"
  $CMD4 > gpurun_out/plain4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_node|k_vin' -s 6 -c 2 -o gpurun_out/prof_${TAG}_cfg4 $CMD4 > gpurun_out/ncu_full4.log 2>&1; echo "ncu full cfg4 rc=$?"
  CMD2="python bench.py --config hh3d_128x128x128 --steps 20 --warmup 3 --no-extra --no-cpu-baseline"
  $CMD2 > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_node' -s 20 -c 1 -o gpurun_out/prof_${TAG}_128 $CMD2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full 128 rc=$?"
fi

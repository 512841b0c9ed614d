cd "${GRAFT_REPO_ROOT:-/root/repo}"
CMD4="python bench.py --steps 3 --warmup 3 --no-extra --no-cpu-baseline"
$CMD4 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_node_pair|k_vin' -s 6 -c 2 -o gpurun_out/prof_r02_v4_cfg4 $CMD4 > gpurun_out/ncu_full4.log 2>&1; echo "ncu full cfg4 rc=$?"

cd "${GRAFT_REPO_ROOT:-/root/repo}"
run() { (cd $1 && timeout 300 python bench.py --config hh3d_512x512x256 --steps 130 --warmup 5 --no-extra --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print("%.4e %.4f ms node %.4f ms frac %.3f" % (d["value"], d["ms_per_step"], r["mean_launch_ms"], r["frac"]))'); }
for rep in 1 2 3; do
  echo "HEAD   $(run .)"
  echo "preaux $(run build_var/pre_aux)"
done

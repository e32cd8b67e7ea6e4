#!/usr/bin/env bash
# Round verification on a B200 (run via gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2700 -- 'bash tools/gpu_check.sh'
# GPU parity tests, smoke, the default bench line, the reference arm, and one full bench
# line (e2e + CPU baselines) per BASELINE config; logs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider \
  > gpurun_out/pytest_gpu.log 2>&1; echo "exit=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2>&1
for c in C1 C2 C3 C3f32 C5; do
  timeout 600 python bench.py --config "$c" > "gpurun_out/bench_$c.json" 2> "gpurun_out/bench_$c.err"
done
timeout 300 python bench.py --config C5 --arith ref --no-e2e --no-cpu > gpurun_out/bench_C5_f32ref.json 2>&1
timeout 300 python bench.py --config C3f32 --arith ref --no-e2e --no-cpu > gpurun_out/bench_C3f32_f32ref.json 2>&1
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], round(d["value"], 2), d["unit"], "T", d["config"].get("temporal_blocking"),
              "e2e", round(d["e2e"]["value"], 1) if d.get("e2e") else None,
              "cpu", round(d["cpu_baseline"]["value"], 3) if d.get("cpu_baseline") else None,
              "clk", d.get("clocks", {}).get("sm_mhz"))
    except Exception as e:
        print(f, "unreadable:", e)
PY

# GPU box: full -m gpu suite, default bench line, Table 1 regime lines.
mkdir -p gpurun_out
python -m paper_2402_08136_b200.build >/dev/null
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; grep "\[parity\]" gpurun_out/pytest_gpu.log | sort | uniq
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; cut -c1-400 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --table1 --steps 20 --warmup 5 --cpu-budget 3 > gpurun_out/bench_table1.jsonl 2> gpurun_out/bench_table1.err
echo "table1 rc=$?"; python - <<'PY'
import json
for l in open("gpurun_out/bench_table1.jsonl"):
    d = json.loads(l); c = d["config"]
    print(c["workload"], c["n_qubits"], "q", round(d["ms_per_step"], 4), "ms  e2e", round(d["e2e"]["seconds"] * 1e3, 3), "ms  launches", d["gpu_launches"], " cpu oracle full", round(d["cpu_baseline"]["extrapolated_full_s"], 3), "s")
PY

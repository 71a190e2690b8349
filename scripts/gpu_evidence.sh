# GPU box: evidence run without profilers -- full -m gpu suite, smoke, bench line, Table 1 lines,
# per-pass profile, virtual-shard scaling projection. (ncu captures go in calls of their own: one
# profiler tool per call.)
python -m paper_2402_08136_b200.build >/dev/null
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --table1 --steps 20 --warmup 5 --cpu-budget 3 > gpurun_out/bench_table1.jsonl 2> gpurun_out/bench_table1.err; echo "table1 rc=$?"
timeout 300 python scripts/pass_profile.py --qpe 1 --kmax 1 --tile 12 --jit 1 --verbose --reps 5 > gpurun_out/pass_profile.txt 2>&1
timeout 900 python scripts/virtual_scaling.py > gpurun_out/virtual_scaling.jsonl 2>&1; echo "virtual rc=$?"
timeout 1200 python scripts/op_microbench.py 30 > gpurun_out/op_microbench.jsonl 2> gpurun_out/op_microbench.err; echo "op micro rc=$?"

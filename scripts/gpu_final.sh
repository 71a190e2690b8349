# GPU box: evidence run -- full -m gpu suite, bench line, Table 1 lines, stress P30, oracle timing,
# per-pass profile, ncu launch list and one ncu --set full capture of the 5 S30 tile passes.
mkdir -p gpurun_out/jit
python -m paper_2402_08136_b200.build >/dev/null
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --table1 --steps 20 --warmup 5 --cpu-budget 3 > gpurun_out/bench_table1.jsonl 2> gpurun_out/bench_table1.err; echo "table1 rc=$?"
timeout 300 python scripts/stress_bench.py --n 30 --kmax 2 > gpurun_out/stress_p30.json 2>&1; echo "stress rc=$?"
timeout 900 python scripts/oracle_timing.py > gpurun_out/oracle_timing.json 2>&1; echo "oracle timing rc=$?"
timeout 300 python scripts/pass_profile.py --qpe 1 --kmax 1 --tile 12 --jit 1 --verbose --reps 5 > gpurun_out/pass_profile.txt 2>&1
# profiler captures: scripts/gpu_profile.sh (launch list) and scripts/gpu_ncu_full.sh (--set full), one call each

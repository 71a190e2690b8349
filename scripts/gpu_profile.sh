# GPU box: per-pass timing and the ncu LAUNCH LIST of the S30 bench step (one profiler tool per call;
# the --set full capture is scripts/gpu_ncu_full.sh, in a call of its own).
mkdir -p gpurun_out
python -m paper_2402_08136_b200.build >/dev/null
timeout 300 python scripts/pass_profile.py --qpe 1 --kmax 1 --tile 12 --jit 1 --verbose --reps 3 > gpurun_out/pass_profile.txt 2>&1
cat gpurun_out/pass_profile.txt
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "ncu rc $?"

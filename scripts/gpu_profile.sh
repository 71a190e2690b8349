# GPU box: per-pass timing, launch list and one ncu --set full capture of the S30 tile passes.
mkdir -p gpurun_out/jit
python -m paper_2402_08136_b200.build >/dev/null
timeout 300 python scripts/pass_profile.py --qpe 1 --kmax 1 --tile 12 --jit 1 --verbose --reps 3 > gpurun_out/pass_profile.txt 2>&1
cat gpurun_out/pass_profile.txt
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
HHLSV_JIT_DUMP=gpurun_out/jit timeout 1500 ncu --set full --clock-control none --import-source on -k regex:hhlsv_tile -c 5 \
  -o gpurun_out/tile_full -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc $?"
ls -la gpurun_out/

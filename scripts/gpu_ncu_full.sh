# GPU box: one ncu --set full capture of the 5 S30 tile passes (the same command first runs without ncu).
mkdir -p gpurun_out/jit
python -m paper_2402_08136_b200.build >/dev/null
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
HHLSV_JIT_DUMP=gpurun_out/jit timeout 1500 ncu --set full --clock-control none --import-source on -k regex:hhlsv_tile -c 5 \
  -o gpurun_out/tile_full -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc $?"

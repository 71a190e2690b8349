# one ncu --set full capture of the 5 S30 tile passes (first program run) + e2e stage profile
set -x
mkdir -p gpurun_out/jit
HHLSV_PROFILE=1 timeout 300 python scripts/e2e_profile.py > gpurun_out/e2e_profile.log 2>&1
HHLSV_JIT_DUMP=gpurun_out/jit timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hhlsv_tile -c 5 \
  -o gpurun_out/tile_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo ncu rc $?

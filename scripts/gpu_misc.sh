# GPU box: e2e stage profile, FP64 microbenchmark, compute-sanitizer (one tool: $SAN_TOOL)
mkdir -p gpurun_out build
python -m paper_2402_08136_b200.build >/dev/null
HHLSV_PROFILE=1 timeout 300 python scripts/e2e_profile.py > gpurun_out/e2e_profile.log 2>&1; tail -40 gpurun_out/e2e_profile.log
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/fp64_peak scripts/microbench/fp64_peak.cu && ./build/fp64_peak | tee gpurun_out/fp64_peak.json
if [ -n "$SAN_TOOL" ]; then
  timeout 1500 compute-sanitizer --tool $SAN_TOOL --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/sanitize_$SAN_TOOL.log 2>&1
  echo "sanitizer $SAN_TOOL rc=$?"; tail -15 gpurun_out/sanitize_$SAN_TOOL.log
fi

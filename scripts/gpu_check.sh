# GPU box: full -m gpu suite (with the [parity] prints) and one default bench line.
mkdir -p gpurun_out
python -m paper_2402_08136_b200.build >/dev/null && python -c "import oracle.sim as s; s.build()" >/dev/null
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log; grep "\[parity\]" gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; cat gpurun_out/bench.json | cut -c1-3000; tail -3 gpurun_out/bench.err

# round profiles: new regression test, launch list of the bench command, ncu --set full of the 5 S30 passes
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k small_tiles 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo launches rc $?
bash scripts/gpu_ncu_full.sh > /dev/null 2>&1; echo full rc $?

for kv in HHLSV_X=0 HHLSV_JIT_NOHOIST=1 HHLSV_JIT_NOCW=1 HHLSV_JIT_NOGROUP=1 HHLSV_JIT_NORTAB=1 HHLSV_JIT_DIRECT=0 HHLSV_JIT_NOPF=1 HHLSV_NO_POOL=1; do
  echo "== $kv $(env $kv timeout 300 python -m pytest tests/test_gpu_parity.py -q -k 'virtual_shards_random' 2>&1 | tail -1)"
done

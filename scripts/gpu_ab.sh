# GPU box: A/B of JIT configurations on the S30 bench step ($AB = space-separated HHLSV_JIT values; "-" = default)
python -m paper_2402_08136_b200.build >/dev/null
for cfg in $AB; do
  [ "$cfg" = "-" ] && cfg=""
  HHLSV_JIT="$cfg" timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err
  python -c "import json; d=json.load(open('/tmp/ab.json')); print(repr('$cfg'), round(d['ms_per_step'],3), 'ms', round(d['roofline']['frac'],4))" || tail -3 /tmp/ab.err
done

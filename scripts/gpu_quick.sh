# quick GPU check: JIT parity tests + bench A/B over an env knob ($AB = "VAR=a VAR=b")
timeout 900 python -m pytest tests -m gpu -x -q -k "jit or hhl or tile or smoke" 2>&1 | tail -4
for kv in $AB; do
  echo "== $kv"; env $kv timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"
done
timeout 300 python scripts/pass_profile.py --qpe 1 --kmax 1 --tile 12 --verbose --reps 3

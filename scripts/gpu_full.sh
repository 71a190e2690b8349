# full GPU suite + e2e stage profile + bench (A/B over $AB)
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
HHLSV_PROFILE=1 timeout 300 python scripts/e2e_profile.py 2>&1 | grep -E "solve|destroy"
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], d['roofline']['frac'], d['e2e'])"

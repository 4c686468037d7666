# re-entry check of the committed tree on a fresh box: GPU tests, smoke, full bench, reference arm
set -x
mkdir -p gpurun_out/check
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/check/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/check/pytest.log
tail -3 gpurun_out/check/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check/smoke.log 2>&1; tail -2 gpurun_out/check/smoke.log
timeout 1500 python bench.py > gpurun_out/check/bench.json 2> gpurun_out/check/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/check/ref_arm.json 2> gpurun_out/check/ref_arm.err; echo "ref rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/check/bench.json').read().strip().splitlines()[-1])
print(json.dumps(d.get('summary'), indent=0))
PY

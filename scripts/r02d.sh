# round-2: whole -m gpu suite, then the bench
set -x
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r02d_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02d_tests.log
python scripts/mm_rep_probe.py
python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r02d_bench.json

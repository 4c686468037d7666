# round-2: full bench (both arms), then the whole -m gpu suite
set -x
nproc; lscpu | grep "Model name"
( time python bench.py --impl reference --steps 5 --warmup 3 ) > gpurun_out/r02c_ref.json 2> gpurun_out/r02c_ref.err
( time python bench.py ) > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
tail -c 3000 gpurun_out/r02c_bench.json
tail -5 gpurun_out/r02c_bench.err
if [ -n "$TESTS" ]; then timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r02c_tests.log 2>&1; tail -5 gpurun_out/r02c_tests.log; fi

# round-1c record: GPU tests, smoke, full bench, headline launch list and
# one --set full capture of the C2 kernel (each ncu command after an
# un-profiled run of the same command)
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01c.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01c.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; echo bench=$?
B="python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline"
$B > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01c.csv $B > /dev/null 2>&1; echo launches=$?
B1="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline"
$B1 > /dev/null 2>&1 && timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:stream_tma_kernel -c 1 -o /tmp/prof_c2_r01c $B1 > /dev/null 2>&1; echo ncu=$?
python scripts/ncu_summary.py /tmp/prof_c2_r01c.ncu-rep > gpurun_out/c2_r01c_summary.md
tail -3 gpurun_out/pytest_gpu_r01c.log

set -x
python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err
B="python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01b.csv $B > /dev/null 2>&1
B1="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline"
$B1 > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:RedqOp -s 3 -c 1 -o gpurun_out/prof_c2_r01b $B1 > /dev/null 2>&1
C3="env C3_REPS=1 C3_BATCH=1 python scripts/c3_sweep.py"
$C3 > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:GfqElemOp -s 2 -c 4 -o gpurun_out/prof_c3_r01b $C3 > /dev/null 2>&1
python scripts/c1_sweep.py > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:PolymulOp -s 30 -c 1 -o gpurun_out/prof_c1_r01b python scripts/c1_sweep.py > /dev/null 2>&1
python scripts/gemv_run.py > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:gfq_gemv_kernel -s 2 -c 2 -o gpurun_out/prof_k5_r01b python scripts/gemv_run.py > /dev/null 2>&1
python scripts/fqt_run.py > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:fqt_conv -c 4 -o gpurun_out/prof_k6_r01b python scripts/fqt_run.py > /dev/null 2>&1
ls gpurun_out/

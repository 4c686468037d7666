set -x
B1="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline"
$B1 > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:RedqOp -s 3 -c 1 -o gpurun_out/prof_c2_r01b $B1 > gpurun_out/ncu_c2.log 2>&1
C3="env C3_REPS=1 C3_BATCH=1 python scripts/c3_sweep.py"
$C3 > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:GfqElemOp -s 2 -c 4 -o gpurun_out/prof_c3_r01b $C3 > gpurun_out/ncu_c3.log 2>&1
python scripts/c1_sweep.py > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:PolymulOp -s 30 -c 1 -o gpurun_out/prof_c1_r01b python scripts/c1_sweep.py > gpurun_out/ncu_c1.log 2>&1
ls gpurun_out/; tail -3 gpurun_out/ncu_c2.log

# round-1 (session 4) re-captures after the C3 dlog table copies and the
# early-staging threshold: launch list of the bench command and --set full of
# the C2 kernel; each command runs once without ncu first
set -x
B="python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01h.csv $B > /dev/null 2>&1
B1="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline"
$B1 > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:stream_tma_kernel -s 3 -c 1 -o gpurun_out/prof_c2_r01h $B1 > /dev/null 2>&1
ls gpurun_out/

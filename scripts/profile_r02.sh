# round-2 ncu captures: launch list of the bench command, then --set full of
# one launch of every headline kernel (each command runs once without ncu first)
set -x
mkdir -p gpurun_out/r02
B="python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches_bench.csv $B > /dev/null 2>&1
run() {  # name kernel-regex skip
    python scripts/prof_one.py $1 > /dev/null 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" -s $3 -c 1 -o gpurun_out/r02/$1 -f python scripts/prof_one.py $1 > gpurun_out/r02/$1.log 2>&1
}
run c2 stream_tma 2
run c1 stream_direct 2
run c3p stream_tma 2
run c3d stream_tma 2
run c3l stream_tma 2
run c4 gfq_matmul_kernel 1
run c5 gfq_matmul_kernel 1
run c5f gfq_matmul_kernel 1
run k5g gfq_gemv_kernel 2
run k5d gfq_gemv_kernel 2
run k6 fqt_mma_kernel 1
ls -la gpurun_out/r02
# summaries on the box (the reports themselves exceed the 64 MiB return limit)
python scripts/ncu_summary.py gpurun_out/r02/*.ncu-rep > gpurun_out/r02/kernels.md 2>&1
for f in gpurun_out/r02/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
du -sh gpurun_out/r02/*
mkdir -p gpurun_out/r02_keep && mv gpurun_out/r02/*.md gpurun_out/r02/*.csv gpurun_out/r02/*.log gpurun_out/r02_keep/ && rm -rf gpurun_out/r02

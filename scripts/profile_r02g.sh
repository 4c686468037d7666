# round-2 final captures of the two kernels that changed after profile_r02.sh
# (C1 direct kernel, C5 K4 with the canonical fold re-pack) and the launch
# list of the bench command; each command runs once without ncu first
set -x
mkdir -p gpurun_out/r02g
B="python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02g/launches_bench.csv $B > /dev/null 2>&1
run() {  # name kernel-regex skip
    python scripts/prof_one.py $1 > /dev/null 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" -s $3 -c 1 -o gpurun_out/r02g/$1 -f python scripts/prof_one.py $1 > gpurun_out/r02g/$1.log 2>&1
}
run c1 stream_direct 2
run c5 gfq_matmul_kernel 1
python scripts/ncu_summary.py gpurun_out/r02g/*.ncu-rep > gpurun_out/r02g/kernels.md 2>&1
for f in gpurun_out/r02g/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
rm -f gpurun_out/r02g/*.ncu-rep
ls -la gpurun_out/r02g

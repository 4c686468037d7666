set -x
for p in 0 1 2; do
ncu --set full --import-source on --clock-control none -k regex:stream_tma --launch-skip 2 -c 1 -o gpurun_out/r02b_c3_p$p -f python scripts/c3_one.py $p > gpurun_out/r02b_ncu_p$p.log 2>&1
done
ls -la gpurun_out

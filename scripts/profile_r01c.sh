# round-1c captures: K4 matmul (C4, C5 with both re-pack modes); each
# command runs once without ncu first
set -x
for spec in "5 redq" "5 fold" "4 redq"; do
  set -- $spec
  M="python scripts/run_matmul.py --cid $1 --reps 1 --repack $2"
  $M > /dev/null 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:gfq_matmul_kernel -c 1 -o gpurun_out/prof_c$1_$2_r01c $M > gpurun_out/ncu_c$1_$2.log 2>&1
done
ls gpurun_out/

# kernel-only durations (ncu gpu__time_duration) of the C1 polymul variants
for l in "" scripts/variants/lib_pm_*.so; do
  echo "== ${l:-in-tree}"
  env ${l:+QPK_DEV_LIB=$l} timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stream_tma_kernel -s 40 -c 5 --csv python scripts/c1_sweep.py 2>/dev/null | grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.]*"' | cut -d, -f3 | tr '\n' ' '; echo
done

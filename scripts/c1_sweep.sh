python scripts/c1_sweep.py
for l in scripts/variants/lib_pm_*.so; do QPK_DEV_LIB=$l python scripts/c1_sweep.py; done

python scripts/c3_sweep.py
for l in scripts/variants/lib_gfe_*.so; do QPK_DEV_LIB=$l python scripts/c3_sweep.py; done

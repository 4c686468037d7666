python scripts/c1_ceiling.py
for l in scripts/variants/lib_*.so; do echo $l; QPK_DEV_LIB=$l python scripts/c1_ceiling.py; done

# round-2 C3 sweep: in-tree library, then every variant under scripts/variants
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$NO_TESTS" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "c3 or gfq_mul or premul_boundary or direct_threshold or fresh_plans" > gpurun_out/r02a_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02a_tests.log
fi
python scripts/c3_sweep.py > gpurun_out/r02a_c3.log 2>&1
for l in scripts/variants/lib_*.so; do QPK_DEV_LIB=$l python scripts/c3_sweep.py >> gpurun_out/r02a_c3.log 2>&1; done
cat gpurun_out/r02a_c3.log

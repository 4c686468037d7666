#!/bin/bash
# Development: build C5 fast-path variants (QPK_MM_EXP=n ...) and print their link paths.
#   scripts/mm_exp.sh TAG "-DQPK_MM_EXP=1"
set -e
cd "$(dirname "$0")/.."
python scripts/build_variant.py "mm3_$1" gfq_matmul_inst_3_v1.o gfq_matmul_inst.cu "-DQPK_INST=3 -DQPK_VARIANT=1 $2"

#!/bin/bash
# A/B of the prefetch-code removal against the previous final build and the round-1 build (3 passes),
# then the GPU tests that touch configuration validation and the bench paths.
cd "$GRAFT_REPO_ROOT"
bash scripts/gpu_variants.sh scripts/var_r02d.txt vd 3 0
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_multiprocess.py -q --timeout 600 -p no:cacheprovider > gpurun_out/m16_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/m16_tests.log

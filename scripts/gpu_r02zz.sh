#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zz.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_apan.py tests/test_gpu_train.py -q -s > gpurun_out/zz_pytest_f34.log 2>&1; echo "rc=$?" >> gpurun_out/zz_pytest_f34.log
grep -E "memory|k=|passed|failed|Error" gpurun_out/zz_pytest_f34.log | tail -16

#!/bin/bash
# compute-sanitizer memcheck over the small GPU tests (fused prep + build, GEMM, write-back, window
# transport loopback, sharded MSPipe-S, staleness error) and racecheck over the teacher-forced tiny
# cases (shared-memory dedup, GEMM stage ring / receive buffers)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
K_MEM="(tiny and (teacher_forced or stream_free_running or multi_step or degenerate or staleness_error or bias_only)) or sampler_edge or abi or (sharded and tiny) or sharded_mitigation"
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -k "$K_MEM" > gpurun_out/memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck.log
tail -4 gpurun_out/memcheck.log
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny and teacher_forced and not bf16" > gpurun_out/racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/racecheck.log
tail -4 gpurun_out/racecheck.log

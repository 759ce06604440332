#!/bin/bash
# round-2 session g: new tests (non-systematic, new codes, run-time specialisation), ablation
OUT=gpurun_out; mkdir -p $OUT
export POLAR_JIT_CACHE=/tmp/polar_jit_r2g
timeout 1500 python -m pytest tests/test_jit.py tests/test_gpu_parity.py -m gpu -x -q -k "jit or specialis or nonsystematic or c2048_1365 or c2048_1536" > $OUT/pytest_r2g.log 2>&1; echo pytest=$?; tail -5 $OUT/pytest_r2g.log
timeout 900 python tools/ablation.py > $OUT/ablation_r2g.jsonl 2> $OUT/ablation_r2g.err; echo ablation=$?; cat $OUT/ablation_r2g.jsonl; tail -3 $OUT/ablation_r2g.err

#!/usr/bin/env bash
# rope/combine rewrite check + checkpoint sweep + B200 latency profile
set -u
OUT=gpurun_out/r1d; mkdir -p $OUT
free -g > $OUT/free.txt; nproc >> $OUT/free.txt
timeout 900 python -m pytest --timeout 300 tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python tools/profile_b200.py --out $OUT/b200_profile.json > $OUT/profile.log 2>&1; echo "rc=$?" >> $OUT/profile.log
timeout 1500 python tools/ckpt_sweep.py --out $OUT/ckpt_sweep.json > $OUT/sweep.log 2>&1; echo "rc=$?" >> $OUT/sweep.log

#!/usr/bin/env bash
# B200 latency profile (reference grid) + checkpoint sweep
set -u
OUT=gpurun_out/r1e; mkdir -p $OUT
timeout 900 python tools/profile_b200.py --out $OUT/b200_profile.json > $OUT/profile.log 2>&1; echo "rc=$?" >> $OUT/profile.log
timeout 1800 python tools/ckpt_sweep.py --out $OUT/ckpt_sweep.json > $OUT/sweep.log 2>&1; echo "rc=$?" >> $OUT/sweep.log

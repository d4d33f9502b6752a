#!/bin/bash
# scratch: packer slice length with the look-back fix-up (bench step and per-layer)
cd /root/repo
mkdir -p gpurun_out
timeout 1500 python tools/ab.py --rounds 1 "rule||" "ts64|GQSA_TARGET_SLOTS=64|" "ts128|GQSA_TARGET_SLOTS=128|" "ts256|GQSA_TARGET_SLOTS=256|" "ts512|GQSA_TARGET_SLOTS=512|" 2>&1 | tee gpurun_out/ab_ts.log

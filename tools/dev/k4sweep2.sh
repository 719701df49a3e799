#!/bin/bash
for b in 50 75 100 125; do for st in 2 3; do
  r=$(DP_DEV_RESIZEP_WARPS=25 DP_DEV_STAGES=$st DP_DEV_RESIZE_PBAND=$b python tools/dev/launchsweep.py resize 16 2>&1 | tail -1)
  echo "band $b stages $st: $r"
done; done
for b in 42 63 84; do
  r=$(DP_DEV_RESIZEP_WARPS=21 DP_DEV_STAGES=3 DP_DEV_RESIZE_PBAND=$b python tools/dev/launchsweep.py resize 16 2>&1 | tail -1)
  echo "w21 band $b: $r"
done

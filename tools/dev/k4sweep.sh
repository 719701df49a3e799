#!/bin/bash
# K4 (periodic taps) knob sweep: consumer warps x stages x band rows.
for w in 21 25 29; do for st in 3 4 5; do for b in 0 2; do
  band=$(( b == 0 ? w : w * b ))
  r=$(DP_DEV_RESIZEP_WARPS=$w DP_DEV_STAGES=$st DP_DEV_RESIZE_PBAND=$band python tools/dev/launchsweep.py resize 16 2>&1 | tail -1)
  echo "warps $w stages $st band $band: $r"
done; done; done

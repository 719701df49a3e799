#!/bin/bash
# Profiling pass for one round (run on the GPU box through gpurun):
#   1. each bench config once WITHOUT ncu (must exit 0 first),
#   2. its launch list (gpu__time_duration, cold-cache, serialised),
#   3. one `ncu --set full` capture of its dominant kernel.
# Outputs under gpurun_out/prof/; summaries are copied into profiles/ by hand.
set -u
out=gpurun_out/prof
mkdir -p $out
declare -A KREGEX=([cfg2]="regex:pipeline_kernel" [cfg3]="regex:roll_kernel" [cfg4]="regex:padded_batches_kernel" [cfg4b]="regex:bucket_rows_batches_kernel" [cfg4r]="regex:ragged_batches_kernel" [cfg1]="regex:range_affine" [cfg5]="regex:pipeline_kernel" [cfg2u8]="regex:gather_copy_kernel" [cfg2rrc]="regex:roll_kernel" [cfg3e]="regex:roll_kernel")
for c in ${CONFIGS:-cfg2 cfg3 cfg5 cfg4 cfg4r cfg4b cfg1 cfg2u8 cfg2rrc cfg3e}; do
  python bench.py --config $c --steps 64 --warmup 32 > $out/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $out/launches_$c.csv \
      python bench.py --config $c --steps 64 --warmup 32 > $out/ncu_list_$c.log 2>&1
  ncu --set full --clock-control none --import-source on -k ${KREGEX[$c]} --launch-skip 4 -c 1 \
      -o $out/full_$c -f python bench.py --config $c --steps 64 --warmup 32 > $out/ncu_full_$c.log 2>&1
  echo "$c done"
done

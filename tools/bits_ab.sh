#!/bin/bash
# bench with bit-packed mask planes (default) vs u8 byte planes on H; R with bits (timed per run)
cd "$(dirname "$0")/.."
for a in "bits_H:" "u8_H:--mask-format u8" "bits_R:--config R"; do
  tag=${a%%:*}; opt=${a#*:}
  s=$(date +%s)
  python bench.py --no-cpu --steps 6 --warmup 3 $opt > gpurun_out/$tag.json 2> gpurun_out/$tag.err
  echo "$tag $(( $(date +%s) - s )) s" >> gpurun_out/bits_times.txt
done

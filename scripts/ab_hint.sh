#!/bin/bash
# A/B: layer lookup by per-warp binary search (old) vs coarse hint table (default).
for c in "--config resnet50" "--config alexnet" "--config lenet" "--config vgg16 --bits 8" "--config 1b --bits 8 --steps 100"; do
  bash scripts/ab.sh ab_hint "$c --no-sgd --no-reduce" old default
done

#!/bin/bash
# A/B: norm-finalize CTA size (it runs beside the unpack on a side stream).
for c in "--config resnet50" "--config alexnet" "--config 1b --bits 8 --steps 100"; do
  bash scripts/ab.sh ab_fin "$c --no-sgd --no-reduce" default fin256 fin128
done

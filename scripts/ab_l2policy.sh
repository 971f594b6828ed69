#!/bin/bash
# A/B: L2 policy of the step's stores — replicas evict-first (default) vs plain (nostcs),
# and the packed stream additionally with an evict_last policy (keep).
for c in "--config alexnet" "--config vgg16 --bits 8" "--config resnet50" "--config 1b --bits 8 --steps 100"; do
  bash scripts/ab.sh ab_l2policy "$c --no-sgd --no-reduce --no-awp-step" nostcs default keep
done

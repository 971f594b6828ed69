#!/bin/bash
# A/B: unpack launched as a programmatic dependent of the pack (default) vs an ordinary launch.
for c in "--config lenet" "--config resnet50" "--config alexnet"; do
  bash scripts/ab.sh ab_pdl "$c --no-sgd --no-reduce" nopdl default
done
python scripts/step_overhead.py

for c in "--config resnet50" "--config alexnet" "--config lenet" "--config vgg16 --bits 8" "--config 1b --bits 24 --steps 100"; do
  bash scripts/ab.sh ab_pers "$c --no-sgd --no-reduce" default pers pers8
done

#!/bin/bash
# Paired A/B on one box: the working tree's csrc ("new") against the files
# saved in ab_base/base/ ("base"), rebuilt on the box in between.
export PYTHONPATH=.
SIZES=${SIZES:-"4096 16384 16384x32768 16384x65536 32768 65536"}
mkdir -p ab_base/new
for f in ab_base/base/*; do cp paper_1111_6549_b200/csrc/$(basename $f) ab_base/new/; done
build() { python -c "from paper_1111_6549_b200 import _lib; _lib.build(force=True)" >/dev/null 2>&1; }
for round in 1 2; do
  echo "== new"; ${CMD:-python scripts/kprobe.py $SIZES}
  cp ab_base/base/* paper_1111_6549_b200/csrc/; build
  echo "== base"; ${CMD:-python scripts/kprobe.py $SIZES}
  cp ab_base/new/* paper_1111_6549_b200/csrc/; build
done

#!/bin/bash
# Build in-tree, then run the given command on B200(s) through gpurun.
# usage: tools/gpu.sh <timeout-seconds> '<command>' [ngpus]
set -e
cd "$(dirname "$0")/.."
make -s -j8 -C paper_2401_08383_b200/csrc 2>&1 | grep -E "error" && { echo "BUILD FAILED"; exit 1; }
make -s -C oracle >/dev/null
exec /usr/local/graft/bin/gpurun --gpus "${3:-1}" --timeout "$1" -- "$2"

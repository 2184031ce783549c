#!/bin/bash
# Build librk.so variants for an A/B run: scripts/ab_build.sh NAME "FLAGS" [NAME "FLAGS" ...] -> alt/NAME.so
set -e
cd "$(dirname "$0")/.."
mkdir -p alt
while [ $# -ge 2 ]; do
  RK_NVCC_FLAGS="$2" python paper_1804_06087_b200/build.py --force > /dev/null
  cp paper_1804_06087_b200/librk.so alt/$1.so
  echo "built alt/$1.so with '$2'"
  shift 2
done
python paper_1804_06087_b200/build.py --force > /dev/null

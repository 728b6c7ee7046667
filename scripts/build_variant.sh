#!/bin/bash
# Build liblob.so from a git revision (or the working tree: WT) into variants/<name>.so
# for A/B timing with LOB_LIB_OVERRIDE.   usage: scripts/build_variant.sh <rev|WT> <name> [extra nvcc flags]
set -e
cd "$(dirname "$0")/.."
rev=$1; name=$2; shift 2
mkdir -p variants
tmp=$(mktemp -d)
if [ "$rev" = "WT" ]; then
  mkdir -p $tmp/paper_2308_13289_b200/csrc $tmp/include
  cp paper_2308_13289_b200/csrc/*.cu paper_2308_13289_b200/csrc/*.cuh $tmp/paper_2308_13289_b200/csrc/
  cp include/lob.h $tmp/include/
else
  git archive $rev paper_2308_13289_b200/csrc include | tar -x -C $tmp
fi
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC,-O2 -shared -DLOB_BUILD_ID="\"variant-$name\"" "$@" -o variants/$name.so $tmp/paper_2308_13289_b200/csrc/lob_api.cu
rm -rf $tmp
echo "variants/$name.so"

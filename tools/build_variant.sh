#!/bin/bash
# Build libradsort.so of another git revision into scratch/ for A/B runs
# (load it with RADSORT_LIB_PATH=$PWD/scratch/libradsort_<name>.so).
#   tools/build_variant.sh <rev> <name>
set -e
cd "$(dirname "$0")/.."
REV=$1; NAME=$2
W=/tmp/radsort_variant_$NAME
rm -rf $W; git worktree prune; git worktree add -f --detach $W $REV > /dev/null
NCCL=$(python -c "import nvidia,os;print(os.path.join(nvidia.__path__[0],'nccl'))")
mkdir -p $W/build scratch
for u in $W/paper_1703_00687_b200/csrc/*.cu; do
  f=$(basename $u .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I "$NCCL/include" \
    -I $W/include -c $u -o $W/build/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scratch/libradsort_$NAME.so $W/build/*.o \
  -L "$NCCL/lib" -l:libnccl.so.2 -Xlinker -rpath="$NCCL/lib"
git worktree remove --force $W
echo scratch/libradsort_$NAME.so

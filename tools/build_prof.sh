#!/bin/bash
# Build scratch/libradsort_prof.so: the library with per-phase clock64 counters
# (-DRADSORT_PHASE_PROF; printed with RADSORT_LOG=1).  Load it with
# RADSORT_LIB_PATH=$PWD/scratch/libradsort_prof.so.  Not used by tests/bench.
set -e
cd "$(dirname "$0")/.."
NCCL=$(python -c "import nvidia,os;print(os.path.join(nvidia.__path__[0],'nccl'))")
mkdir -p build/prof scratch
for u in paper_1703_00687_b200/csrc/*.cu; do
  f=$(basename $u .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DRADSORT_PHASE_PROF \
    -I "$NCCL/include" -c paper_1703_00687_b200/csrc/$f.cu -o build/prof/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scratch/libradsort_prof.so build/prof/*.o \
  -L "$NCCL/lib" -l:libnccl.so.2 -Xlinker -rpath="$NCCL/lib"

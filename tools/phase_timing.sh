#!/bin/bash
# Build a phase-timing variant of libgbxcu (-DGBX_PHASE_TIMING) into tools/timing/
# and print per-phase cycle shares of the train kernel (CTA 0) for a few batch sizes.
set -e
D=tools/timing; mkdir -p $D
ARCH="-gencode arch=compute_100a,code=sm_100a"
NCCL=$(python3 -c "import nvidia.nccl as m; print(list(m.__path__)[0])")
for f in gbxcu_api k_forward k_train k_train_tc k_train_cl k_shuffle k_aggregate k_wide k_wide16 k_qtable; do
  nvcc $ARCH -O3 -std=c++17 -Xcompiler -fPIC -DGBX_PHASE_TIMING -Ipaper_2111_12055_b200/csrc -Iinclude -I$NCCL/include -c paper_2111_12055_b200/csrc/$f.cu -o $D/$f.o &
done; wait
nvcc $ARCH -shared -o $D/libgbxcu.so $D/*.o -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker $NCCL/lib -lcudart

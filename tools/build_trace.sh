#!/bin/bash
# Debug build with the GRU phase trace compiled in: tools/libddppo_trace.so
set -e
cd "$(dirname "$0")/.."
SRC=paper_1911_00357_b200/csrc
ND=$(python -c "import paper_1911_00357_b200.build as b; print(b.nccl_dir())")
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -DDDPPO_TRACE -shared \
  -I include -o tools/libddppo_trace.so $SRC/*.cu -L$ND -l:libnccl.so.2 -Xlinker -rpath,$ND

#!/bin/bash
# Debug builds with phase traces compiled in: tools/libddppo_trace.so (GRU recurrence, tools/trace_gru.py)
# and tools/libddppo_tctrace.so (TMA conv kernel, tools/trace_tconv.py)
set -e
cd "$(dirname "$0")/.."
SRC=paper_1911_00357_b200/csrc
ND=$(python -c "import paper_1911_00357_b200.build as b; print(b.nccl_dir())")
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -DDDPPO_TRACE -shared \
  -I include -o tools/libddppo_trace.so $SRC/*.cu -L$ND -l:libnccl.so.2 -Xlinker -rpath,$ND
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -DDDPPO_TCONV_TRACE -shared \
  -I include -o tools/libddppo_tctrace.so $SRC/*.cu -L$ND -l:libnccl.so.2 -Xlinker -rpath,$ND

#!/bin/bash
# Build the diagnostics library librwb_trace.so (-DRWB_TRACE) next to librwb.so
# (RWB_TRACE_EXTRA: more -D flags, e.g. -DRWB_EXP_NOTMEM for the SpMV-without-TMEM experiment).
cd "$(dirname "$0")/.." || exit 1
C=paper_2509_26213_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -DRWB_TRACE $RWB_TRACE_EXTRA -I include -o paper_2509_26213_b200/_lib/librwb_trace.so \
  $C/rwb_ops.cu $C/rwb_solve.cu $C/rwb_resident.cu $C/rwb_resident4.cu $C/rwb_resident2d.cu $C/rwb_chunks.cu $C/rwb_mgcg.cu $C/rwb_render.cu

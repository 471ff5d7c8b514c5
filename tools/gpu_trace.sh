#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_cs_0412107_b200/libmcinv.so
cp ab/libmcinv_trace.so $L
timeout 300 python tools/trace_v6.py gpurun_out/trace.bin > gpurun_out/trace.log 2>&1; echo "rc=$?" >> gpurun_out/trace.log

#!/bin/bash
# config-2 A/B timings of library variants (ab/libmcinv_<v>.so, tools/ab_variant.sh), each
# entry "<variant>[:VAR=value,...]" (runtime knobs); timing only
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_cs_0412107_b200/libmcinv.so
cp $L /tmp/libmcinv_prod.so
OUT=gpurun_out/${ABL_OUT:-abl.log}
: > $OUT
for e in ${ABL_LIST:-base}; do
  v=${e%%:*}; envs=""; [ "$v" != "$e" ] && envs=$(echo ${e#*:} | tr ',' ' ')
  cp ab/libmcinv_$v.so $L
  echo "== $e" >> $OUT
  env $envs timeout 120 python tools/run_one.py --config ${ABL_CFG:-2} --sweeps ${ABL_SWEEPS:-220} --burn ${ABL_BURN:-20} --repeat 2 ${ABL_ARGS:-} >> $OUT 2>&1; echo "rc=$?" >> $OUT
done
cp /tmp/libmcinv_prod.so $L
[ -n "$ABL_TRACE" ] && { cp ab/libmcinv_trace.so $L; env $ABL_TRACE timeout 300 python tools/trace_v6.py gpurun_out/trace.bin > gpurun_out/trace.log 2>&1; cp /tmp/libmcinv_prod.so $L; }
true

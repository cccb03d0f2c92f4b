#!/bin/bash
# Fused-pass DRAM traffic and duration per launch vs cluster shape / z-chunk (ncu launch metrics
# of the fused launches of one C4 512^3 step with fused passes up to k = 30).
#   VARIANTS="none:64 2x4:64 ..." bash tools/fused_zc.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python tools/prof_step.py 512 1 1 30 > gpurun_out/zc_plain.log 2>&1 || { tail -5 gpurun_out/zc_plain.log; exit 1; }
for V in ${VARIANTS:-none:64 2x2:64 2x4:64 2x4p0:64 none:512}; do
  CL=${V%%:*}; ZC=${V##*:}; PS=1
  case $CL in *p0) PS=0; CL=${CL%p0};; esac
  [ "$CL" = none ] && CL=""
  PSP_FUSED_VERBOSE=1 PSP_FUSED_CL=$CL PSP_FUSED_PSYNC=$PS PSP_FUSED_ZC=$ZC timeout 900 ncu \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:fused_tma --csv --log-file gpurun_out/zc_$V.csv \
    python tools/prof_step.py 512 1 1 30 > gpurun_out/zc_$V.log 2>&1
  echo "variant $V rc $?"
done

#!/bin/bash
# DRAM bytes of a few fused launches (k ~ 10..13 of the first cycle) per cluster variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python tools/prof_step.py 512 1 1 16 > gpurun_out/fd_plain.log 2>&1 || { tail -5 gpurun_out/fd_plain.log; exit 1; }
for CL in ${CLS:-none 2x4 1x2}; do
  C=$CL; [ "$C" = none ] && C=""
  PSP_FUSED_CL=$C timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum \
    --clock-control none -k regex:fused_tma -s 9 -c 3 --csv --log-file gpurun_out/fd_$CL.csv \
    python tools/prof_step.py 512 1 1 16 > gpurun_out/fd_$CL.log 2>&1
  echo "variant $CL rc $?"
done

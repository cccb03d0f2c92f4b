cd "${GRAFT_REPO_ROOT:-/root/repo}"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-c5"
$CMD > gpurun_out/b1.json 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_r01c.csv $CMD > gpurun_out/ncu_b1.log 2>&1
python tools/kbench.py matvec 512 10
echo done

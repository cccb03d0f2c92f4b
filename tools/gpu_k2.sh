cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
python tools/kbench.py matvec 512 20
python tools/kbench.py matvec 512 3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:march -s 1 -c 1 -o gpurun_out/prof_matvec2 python tools/kbench.py matvec 512 3 > gpurun_out/ncu_matvec2.log 2>&1
tail -1 gpurun_out/ncu_matvec2.log

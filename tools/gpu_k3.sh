cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; tail -15 gpurun_out/pytest_gpu.log
python tools/kbench.py matvec 512 20
PSP_LIB=build/v3/libpspgmres.so python tools/kbench.py matvec 512 20
for d in 1 3 4; do timeout 120 python tools/kbench.py mrep 27 32 $d 3; done

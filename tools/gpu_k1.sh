cd "${GRAFT_REPO_ROOT:-/root/repo}"
python tools/kbench.py matvec 512 20 > gpurun_out/kb_matvec.txt 2>&1
python tools/kbench.py mrep 27 32 3 3 > gpurun_out/kb_mrep.txt 2>&1
for d in 1 2 3 4; do python tools/kbench.py solve 27 $d 10; done > gpurun_out/kb_solve.txt 2>&1
cat gpurun_out/kb_*.txt
python tools/kbench.py matvec 512 3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:march -s 1 -c 1 -o gpurun_out/prof_matvec python tools/kbench.py matvec 512 3 > gpurun_out/ncu_matvec.log 2>&1
tail -3 gpurun_out/ncu_matvec.log

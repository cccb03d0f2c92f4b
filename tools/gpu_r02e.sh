#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02e
mkdir -p $O
for i in 1 2; do
  python tools/kbench.py matvec 512 20 > $O/mv2_$i.txt 2>&1
  PSP_MARCH4_MINB=3 python tools/kbench.py matvec 512 20 > $O/mv3_$i.txt 2>&1
done
for d in 1 2 3 4; do python tools/kbench.py solve 26 $d 10 > $O/solve$d.txt 2>&1; done
python tools/cfg_step.py c1 5 1 2 > $O/c1.txt 2>&1
python tools/cfg_step.py c2 20 1 2 > $O/c2.txt 2>&1
head -50 $O/*.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -25 $O/pytest.log

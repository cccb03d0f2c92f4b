#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r02d
mkdir -p $O
timeout 300 python tools/debug_slabs.py C2s fused 2 > $O/dbg_c2s.txt 2>&1; tail -50 $O/dbg_c2s.txt
timeout 300 python tools/debug_slabs.py C4s fused 2 > $O/dbg_c4s.txt 2>&1; tail -8 $O/dbg_c4s.txt
python tools/kbench.py mrep 27 32 3 3 > $O/kb_mrep.txt 2>&1; python tools/kbench.py mrep 26 32 2 3 >> $O/kb_mrep.txt 2>&1
python tools/kbench.py mrep 26 32 4 3 >> $O/kb_mrep.txt 2>&1; PSP_MREP_SPLIT=1 python tools/kbench.py mrep 27 32 3 3 >> $O/kb_mrep.txt 2>&1
cat $O/kb_mrep.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -25 $O/pytest.log

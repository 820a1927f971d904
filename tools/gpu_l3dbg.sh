#!/bin/bash
O=gpurun_out/l3dbg; mkdir -p $O
FFDP_NO_TMA=1 timeout 120 python tools/l3dbg.py > $O/notma.log 2>&1; echo rc=$? >> $O/notma.log
timeout 120 python tools/l3dbg.py > $O/tma.log 2>&1; echo rc=$? >> $O/tma.log
timeout 300 compute-sanitizer --tool memcheck python tools/l3dbg.py > $O/san.log 2>&1; echo rc=$? >> $O/san.log
tail -5 $O/notma.log $O/tma.log; grep -m 20 -i "error\|invalid\|illegal\|at 0x\|by thread" $O/san.log

#!/bin/bash
O=gpurun_out/${1:-localdbg}; mkdir -p $O
timeout 120 python -X faulthandler -c "
import faulthandler, sys, runpy
faulthandler.dump_traceback_later(90, exit=True)
sys.argv=['bench.py','--gpus','2','--transport','local','--workload','mi256','--steps','5','--warmup','3']
runpy.run_path('bench.py', run_name='__main__')
" > $O/out.json 2> $O/err.log; echo "rc=$?" >> $O/err.log
tail -60 $O/err.log; cat $O/out.json | head -c 600

timeout 900 python -X faulthandler -c "
import sys, runpy, traceback
sys.argv=['bench.py','--strong','--layout','cols','--steps','50','--warmup','3','--no-c5-extra','--skip-e2e']
import bench
args=bench.parse_args(sys.argv[1:])
import os
os.environ.setdefault('MASTER_ADDR','127.0.0.1'); os.environ.setdefault('MASTER_PORT','29533')
import torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group('nccl', rank=0, world_size=1)
try:
    r = bench.run_strong(args, bench.CONFIGS['c2'], 0, 1, 0)
    print('returned', r, file=sys.stderr)
except BaseException as e:
    traceback.print_exc()
    print('EXC', repr(e), file=sys.stderr)
" > gpurun_out/r02_dbg.out 2> gpurun_out/r02_dbg.err; echo "rc=$?"
grep -v "Warning\|return func" gpurun_out/r02_dbg.err | tail -n 30; head -c 300 gpurun_out/r02_dbg.out

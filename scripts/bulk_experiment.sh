cat > /tmp/bulk_parity.py <<'PY'
import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
import gpu_util as U
from paper_2303_06324_b200 import occl
from oracle import ring
comms = occl.local_group(8, 0, gridBlocks=18, sliceBytes=192 << 10, stagingTiles=5, maxColl=16, bulkStores=1)
for ci, (kind, dtype, count) in enumerate([("allreduce", "f32", 3_000_017), ("allreduce", "bf16", 2_500_003),
                                           ("allgather", "f32", 400_009), ("reducescatter", "bf16", 300_007),
                                           ("broadcast", "f32", 2_000_001), ("allreduce", "i32", 1 << 22)]):
    sends, recvs = U.make_bufs(kind, dtype, 8, count, 40 + ci, ci)
    U.run_collective(comms, kind, sends, recvs, ci, count, dtype, 3)
    U.check_full(kind, dtype, 8, count, 40 + ci, ci, recvs, 3)
    print("ok", kind, dtype, flush=True)
occl.destroy_group(comms)
PY
timeout -s KILL 300 python /tmp/bulk_parity.py 2>&1 | tail -8
timeout -s KILL 400 bash scripts/sweep_cfgs.sh scripts/sweep15.txt

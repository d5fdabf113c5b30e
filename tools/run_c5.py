"""Run config c5 (or a smaller hex8 config) through the row-partitioned path.
  python tools/run_c5.py [--config c5] [--world W] [--snapshots 48]
Under torchrun (WORLD_SIZE > 1): one partition per rank over NCCL."""
import argparse, json, os, sys
sys.path.insert(0, '.')
from paper_2207_02543_b200 import c5

ap = argparse.ArgumentParser()
ap.add_argument('--config', default='c5')
ap.add_argument('--world', type=int, default=1)
ap.add_argument('--snapshots', type=int, default=48)
ap.add_argument('--batch', type=int, default=8)
ap.add_argument('--k', type=int, default=None)
a = ap.parse_args()
ws = int(os.environ.get('WORLD_SIZE', '1'))
if ws > 1:
    import torch, torch.distributed as dist
    rank = int(os.environ['RANK']); torch.cuda.set_device(int(os.environ['LOCAL_RANK']))
    dist.init_process_group('nccl')
    from paper_2207_02543_b200.partition import PartitionedSolver
    uid = [PartitionedSolver.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    res, _ = c5.run(a.config, ws, [rank], uid[0], a.snapshots, a.batch, a.k,
                    device=int(os.environ['LOCAL_RANK']))
else:
    res, _ = c5.run(a.config, a.world, None, None, a.snapshots, a.batch, a.k)
res.pop('history')
print(json.dumps(res))

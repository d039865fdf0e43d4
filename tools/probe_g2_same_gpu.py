import os, sys, torch, torch.distributed as dist
sys.path.insert(0, '/root/repo')
import paper_2603_23198_b200 as sffn
rank = int(os.environ['RANK']); world = int(os.environ['WORLD_SIZE'])
torch.cuda.set_device(0)
dist.init_process_group('gloo')
try:
    c = sffn.Comm(rank, world, 0)
    print('rank', rank, 'comm ok', flush=True)
except Exception as e:
    print('rank', rank, 'comm failed:', e, flush=True)

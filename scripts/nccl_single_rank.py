"""ShardedDSG + TorchComm over NCCL with one rank (the NCCL code path of the
multi-GPU denoiser on a one-GPU box; development aid).  Run under torchrun:
python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1
scripts/nccl_single_rank.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import torch.distributed as dist

import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200.parallel import ShardedDSG, TorchComm

dist.init_process_group("nccl")
torch.cuda.set_device(0)
n = 1024
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(n, n, device="cuda", generator=g)
sh = ShardedDSG(p, n, n, 1, [0], TorchComm(), device=torch.device("cuda", 0))
sh.load(x)
sh.denoise()
out = sh.gather()
ref = pnp.dsg_nlm_denoise(x, p)
print("nccl single-rank sharded == single:", torch.equal(out, ref), flush=True)
dist.destroy_process_group()

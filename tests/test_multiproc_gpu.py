"""The row-strip sharded algorithm run by two real processes (torch.distributed
world size 2, gloo, messages staged through host memory: parallel.
HostStagedComm), both on cuda:0 -- every exchange completes on the host
before the next launch, so no rank's kernels wait on the other's.  The
gathered strips must equal the single-GPU call bit for bit: the adaptive
denoise (ShardedDSG.denoise) and the frozen-guide SR ADMM
(ShardedSRADMM.freeze + run), on the P-templated and the general sweep."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, job, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1901_06110_b200 as pnp
        from paper_1901_06110_b200.parallel import HostStagedComm, ShardedDSG, ShardedSRADMM
        dev = torch.device("cuda", 0)
        kind = job["kind"]
        p = pnp.PatchParams(*job["params"])
        if kind == "dsg":
            x = torch.from_numpy(job["x"]).to(dev)
            H, W = x.shape
            sh = ShardedDSG(p, H, W, world, [rank], HostStagedComm(), device=dev)
            sh.load(x)
            sh.denoise()
            y0, y1 = sh.states[0].lay.rows
            q.put((rank, y0, y1, sh.states[0].own(sh.states[0].out).cpu().numpy(), None))
        else:
            op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
            guide = torch.from_numpy(job["guide"]).to(dev)
            H, W = guide.shape
            sh = ShardedSRADMM(op, p, H, W, world, [rank], HostStagedComm(), device=dev)
            sh.load(torch.from_numpy(job["y"]).to(dev), guide, torch.from_numpy(job["truth"]).to(dev))
            sh.freeze()
            cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=job["iters"],
                                   constraint=pnp.UNIT_BOX)
            recs = sh.run(cfg)
            e = sh.st[rank]
            y0, y1 = e["rows"]
            q.put((rank, y0, y1, sh.gather().cpu().numpy(), np.array(recs)))
    finally:
        dist.destroy_process_group()


def _run_world2(job):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, job, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    return sorted(res, key=lambda t: t[0])


@pytest.mark.parametrize("params", [(7, 10, 0.1, 2.0), (17, 21, 0.15, None)])
def test_two_process_sharded_denoise_bitwise(params):
    import paper_1901_06110_b200 as pnp
    rng = np.random.default_rng(31)
    x = rng.random((416, 200)).astype(np.float32)
    res = _run_world2({"kind": "dsg", "params": params, "x": x})
    ref = pnp.dsg_nlm_denoise(torch.from_numpy(x).cuda(), pnp.PatchParams(*params)).cpu().numpy()
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == x.shape[0]
    got = np.concatenate([r[3] for r in res], axis=0)
    assert np.array_equal(got, ref)


def test_two_process_sharded_sr_admm_bitwise():
    import paper_1901_06110_b200 as pnp
    g = torch.Generator(device="cuda").manual_seed(32)
    H, W = 312, 200
    truth = torch.rand(H, W, device="cuda", generator=g)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    y = (op.apply_device(truth) + 0.02 * torch.randn(H // 2, W // 2, device="cuda",
                                                       generator=g)).contiguous()
    guide = (truth + 0.05 * torch.randn(H, W, device="cuda", generator=g)).clamp(0, 1)
    params = (7, 10, 0.1, 1.5)
    iters = 5
    res = _run_world2({"kind": "sr", "params": params, "guide": guide.cpu().numpy(),
                       "y": y.cpu().numpy(), "truth": truth.cpu().numpy(), "iters": iters})
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=iters,
                           constraint=pnp.UNIT_BOX)
    prob = pnp.make_sr_problem(op, y, ground_truth=truth)
    v1, recs = pnp.linearized_pnp_admm(
        prob, cfg, denoiser=pnp.freeze_guide(guide, pnp.PatchParams(*params)).as_denoiser())
    got = np.concatenate([r[3] for r in res], axis=0)
    assert np.array_equal(got, v1.cpu().numpy())
    ref = np.array([[r.index, r.primal, r.dual, r.psnr, r.objective] for r in recs])
    for r in res:  # every rank holds the all-reduced records
        assert np.allclose(r[4], ref, rtol=1e-9, atol=0)

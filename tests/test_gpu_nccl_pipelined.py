"""The bench's N-GPU step shape on one GPU: an NCCL process group of size 1, the per-sample outputs gathered
with gather_outputs inside SafetyFilter.solve_pipelined's finish hook (NCCL collectives issued from the side
streams, two batches in flight).  Exercises the stream / collective interplay the driver's multi-GPU bench runs;
with one rank the gather is an identity, so the results must equal solve_batched's."""
import os

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("asynchronous", [False, True])
def test_pipelined_solve_with_nccl_gather_world1(asynchronous):
    import torch.distributed as dist

    from paper_2501_19042_b200 import SafetyFilter, SolverConfig, sample_proposals
    from paper_2501_19042_b200.distributed import gather_outputs, gather_outputs_async
    from paper_2501_19042_b200.scenarios import config_problem
    import socket
    with socket.socket() as sk:   # a free port (127.0.0.1 rendezvous)
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        prob = config_problem(2)
        cfg = SolverConfig(max_iters=100, svars=False)
        sf = SafetyFilter(prob, degree=10, config=cfg)
        xs = [torch.from_numpy(sample_proposals(prob, sf.basis, 200, seed=s).proposals).cuda() for s in range(4)]
        gathered = {}

        def finish(k, out):
            if asynchronous:   # (the bench's N-GPU step: collectives not waited for on the batch's stream)
                gathered[k] = gather_outputs_async(out, out.coeffs.shape[0])
            else:
                gathered[k] = gather_outputs(out, out.coeffs.shape[0])

        outs = sf.solve_pipelined(iter(xs), config=cfg, finish=finish)
        if asynchronous:
            for k in list(gathered):
                gathered[k] = gathered[k]()
        torch.cuda.synchronize()
        for k, x in enumerate(xs):
            ref = sf.solve_batched(x, config=cfg)
            assert torch.equal(gathered[k]["coeffs"], ref.coeffs)
            assert torch.equal(gathered[k]["iterations"], ref.iterations)
            assert torch.equal(outs[k].feasible, ref.feasible)
    finally:
        dist.destroy_process_group()

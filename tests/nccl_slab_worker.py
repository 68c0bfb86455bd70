"""Worker of tests/test_gpu_nccl.py: one rank of a z-slab solve over the library's NCCL transport
(csrc/comm.cpp NcclTransport: ncclSend/Recv halo planes, AllReduce of the owned norms, AllGather of
the coarse right-hand side).  Launched by torch.distributed.run, one process
per GPU.  Every rank also solves the whole problem on its own GPU with a one-rank context and
compares its slab with it: operators change no arithmetic of any point, so the V-cycle must agree
bitwise and the solve to 1e-12 with the same cycle count (the same bar as the loopback tests in
tests/test_gpu_multirank.py).  Prints "NCCL_SLAB_OK rank r" on success; any mismatch raises."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pmg_inputs as pi  # noqa: E402
import paper_1808_03595_b200 as pmg  # noqa: E402

CASES = [
    dict(k=(3, 2, 5), p=4, lam=1.7, stretch=1.4),
    dict(k=(3, 3, 4), p=8, lam=0.0, stretch=None),
    dict(k=(2, 2, 4), p=12, lam=0.0, stretch=1.2),
]


def main():
    rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    for cfg in CASES:
        case = pi.small_case(cfg["k"], cfg["p"], cfg["lam"], stretch=cfg["stretch"])
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(pmg.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())

        # the whole problem on this rank's GPU (one-rank context)
        s1 = pmg.Solver(case.k, case.widths, case.p, case.lam)
        x = [s1.grid_coords(s1.nlevels - 1, d) for d in range(3)]
        f_np = case.f_nodal(x)
        F1 = s1.new_grid()
        s1.weak_rhs(torch.from_numpy(f_np).cuda(), F1)
        u1 = s1.new_grid()
        rep1 = s1.solve(F1, u1, 1e-10)
        torch.cuda.synchronize()
        F_np, u1 = F1.cpu().numpy(), u1.cpu().numpy()
        s1.close()

        # this rank's z-slab over NCCL
        s = pmg.Solver(case.k, case.widths, case.p, case.lam, rank=rank, nranks=ws, nccl_id=nccl_id)
        sl = s.slab
        pl = (case.k[0] * case.p + 1) * (case.k[1] * case.p + 1)
        lo, hi = sl["z0"] * case.p * pl, (sl["z1"] * case.p + 1) * pl
        F_loc = s.new_grid()
        s.weak_rhs(torch.from_numpy(f_np[lo:hi].copy()).cuda(), F_loc)
        torch.cuda.synchronize()
        assert np.array_equal(F_loc.cpu().numpy(), F_np[lo:hi]), "slab weak RHS differs"
        u = s.new_grid()
        rep = s.solve(F_loc, u, 1e-10)
        torch.cuda.synchronize()
        assert rep["cycles"] == rep1["cycles"], (rep["cycles"], rep1["cycles"])
        err = np.abs(u.cpu().numpy() - u1[lo:hi]).max() / np.abs(u1).max()
        assert err <= 1e-12, (cfg, err)
        s.close()
        dist.barrier()
    print("NCCL_SLAB_OK rank %d" % rank, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

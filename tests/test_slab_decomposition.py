"""z-slab decomposition on the CPU.

1. The library's plan (pmg_slab_plan, pure host arithmetic of libpmg.so) partitions the record
   planes: every global plane is owned by exactly one rank.
2. Dependency footprints, checked with the ORACLE's operators: each operator's values on a rank's
   owned record planes depend only on inputs inside the rank's local planes [zb, z1] (ghosts
   included) -- the halo depth the CUDA path exchanges is sufficient.
3. world_size 2 and 3 gloo process groups replay the library's exchange pattern (halo planes,
   the one-directional grid shift for the condensation, the allgather of the coarse right-hand
   side, the allreduce of owned dot products) with the plan's offsets and check the result
   against the undivided vector.
"""
import os
import socket

import numpy as np
import pytest

import pmg_inputs as pi

pmg = pytest.importorskip("paper_1808_03595_b200")


def test_plan_partitions_planes():
    for k3 in range(1, 21):
        for nr in range(1, min(k3, 8) + 1):
            owned = []
            for r in range(nr):
                s = pmg.slab_plan(k3, nr, r)
                assert s["z0"] < s["z1"]
                assert s["nplanes"] == s["z1"] - s["zb"] + 1
                assert s["zb"] == max(s["z0"] - 1, 0)
                owned += [s["zb"] + q for q in range(s["own_lo"], s["own_hi"])]
                assert (s["lower"] == r - 1) if r > 0 else s["lower"] == -1
                assert (s["upper"] == r + 1) if r < nr - 1 else s["upper"] == -1
            assert sorted(owned) == list(range(k3 + 1)), (k3, nr)


def test_plan_rejects_bad_input():
    with pytest.raises(pmg.PmgError):
        pmg.slab_plan(2, 3, 0)          # k3 < nranks
    with pytest.raises(pmg.PmgError):
        pmg.slab_plan(8, 2, 2)          # rank out of range


# ---------------------------------------------------------------- footprints (oracle)
def _record_plane(mesh):
    """record plane of every global grid point: v3 = i3 // p."""
    i3 = mesh.idx[2].ravel()
    return i3 // mesh.p


@pytest.mark.parametrize("nr", [2, 3])
def test_footprints_match_halo_depth(nr):
    from oracle import condensed, mg
    case = pi.small_case((2, 2, 5), 4, 0.7, stretch=1.3)
    H = mg.Hierarchy(case.k, case.widths, case.p, case.lam, coarse_rtol=1e-13)
    fine, coarse = H.levels[-1], H.levels[-2]
    rng = np.random.default_rng(5)
    mf, mc = fine.mesh, coarse.mesh
    vf, vc = _record_plane(mf), _record_plane(mc)
    i3f = mf.idx[2].ravel()
    for r in range(nr):
        s = pmg.slab_plan(case.k[2], nr, r)
        own_f = (vf >= s["zb"] + s["own_lo"]) & (vf < s["zb"] + s["own_hi"])
        own_c = (vc >= s["zb"] + s["own_lo"]) & (vc < s["zb"] + s["own_hi"])
        outside_f = (vf < s["zb"]) | (vf > s["z1"])
        outside_c = (vc < s["zb"]) | (vc > s["z1"])

        def perturbed(x, outside):
            y = x.copy()
            y[outside] += rng.standard_normal(int(outside.sum()))
            return y

        u = rng.standard_normal(mf.ntot) * mf.free_skel
        f = rng.standard_normal(mf.ntot) * mf.free_skel
        # residual: owned values see u only on the local planes
        a = fine.op.residual(u, f)
        b = fine.op.residual(perturbed(u, outside_f) * mf.free_skel, f)
        assert np.array_equal(a[own_f], b[own_f])
        # smoother: owned corrections see r only on the local planes
        a = fine.smoother.apply(f)
        b = fine.smoother.apply(perturbed(f, outside_f) * mf.free_skel)
        assert np.allclose(a[own_f], b[own_f], rtol=0, atol=1e-13 * np.abs(a).max())
        if s["lower"] >= 0:   # and the ghost plane below is really needed (the halo is not too deep)
            ghost_f = vf == s["zb"]
            b = fine.op.residual(perturbed(u, ghost_f) * mf.free_skel, f)
            a2 = fine.op.residual(u, f)
            assert np.abs(a2[own_f] - b[own_f]).max() > 1e-6
            b = fine.smoother.apply(perturbed(f, ghost_f) * mf.free_skel)
            assert np.abs(fine.smoother.apply(f)[own_f] - b[own_f]).max() > 1e-6
        # restriction: owned coarse values see fine r only on the local planes
        T = H.transfers[-1]
        a = T.restrict(f)
        b = T.restrict(perturbed(f, outside_f) * mf.free_skel)
        assert np.allclose(a[own_c], b[own_c], rtol=0, atol=1e-13 * np.abs(a).max())
        # prolongation: owned fine values see coarse u only on the local planes
        uc = rng.standard_normal(mc.ntot) * mc.free_skel
        a = T.prolong(uc)
        b = T.prolong(perturbed(uc, outside_c) * mc.free_skel)
        assert np.array_equal(a[own_f], b[own_f])
        # condensation: owned values see the grid RHS only on planes zb p .. z1 p (ghost element)
        F = rng.standard_normal(mf.ntot)
        out_grid = (i3f < s["zb"] * mf.p) | (i3f > s["z1"] * mf.p)
        a = fine.op.condense(F)
        b = fine.op.condense(perturbed(F, out_grid))
        assert np.allclose(a[own_f], b[own_f], rtol=0, atol=1e-13 * np.abs(a).max())


# ---------------------------------------------------------------- gloo replay of the exchanges
def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, k3, plane, p, nx, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1808_03595_b200 as lib
        s = lib.slab_plan(k3, world, rank)
        plans = [lib.slab_plan(k3, world, r) for r in range(world)]
        g = torch.from_numpy(np.random.default_rng(3).standard_normal((k3 + 1, plane)))
        g[k3] = 0.0                                         # Dirichlet top plane
        zb, z1 = s["zb"], s["z1"]
        loc = g[zb:z1 + 1].clone()
        ghost = torch.ones(loc.shape[0], dtype=torch.bool)
        ghost[s["own_lo"]:s["own_hi"]] = False
        loc[ghost] = float("nan")
        # halo: own_lo -> lower's top plane, own_hi - 1 -> upper's plane 0 (pmg.h, comm.cpp halo())
        reqs = []
        if s["lower"] >= 0:
            reqs.append(dist.isend(loc[s["own_lo"]].clone(), s["lower"]))
            reqs.append(dist.irecv(loc[0], s["lower"]))
        if s["upper"] >= 0:
            reqs.append(dist.isend(loc[s["own_hi"] - 1].clone(), s["upper"]))
            reqs.append(dist.irecv(loc[-1], s["upper"]))
        for rq in reqs:
            rq.wait()
        assert torch.equal(loc, g[zb:z1 + 1]), "halo exchange"
        # owned dot products summed over ranks
        t = (loc[s["own_lo"]:s["own_hi"]] ** 2).sum().reshape(1)
        dist.all_reduce(t)
        assert abs(t.item() - (g ** 2).sum().item()) <= 1e-12 * (g ** 2).sum().item()
        # allgather of the owned planes, padded to the largest owned count, then placed at z0
        chunk = max(P["own_hi"] - P["own_lo"] for P in plans) * plane
        send = torch.zeros(chunk, dtype=torch.float64)
        own = loc[s["own_lo"]:s["own_hi"]].reshape(-1)
        send[:own.numel()] = own
        recv = [torch.zeros(chunk, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(recv, send)
        full = torch.full_like(g, float("nan"))
        for r, P in enumerate(plans):
            cnt = P["own_hi"] - P["own_lo"]
            full[P["z0"]:P["z0"] + cnt] = recv[r][:cnt * plane].reshape(cnt, plane)
        assert torch.equal(full, g), "coarse allgather"
        # grid shift for the condensation: p planes below the top plane go to the upper rank
        ng = torch.from_numpy(np.random.default_rng(4).standard_normal((k3 * p + 1, nx)))
        mine = ng[s["z0"] * p: s["z1"] * p + 1]                 # the caller's slab
        locg = torch.full(((z1 - zb) * p + 1, nx), float("nan"), dtype=torch.float64)
        gh = (s["z0"] - zb) * p
        locg[gh:] = mine
        reqs = []
        if s["upper"] >= 0:
            reqs.append(dist.isend(locg[-1 - p:-1].clone(), s["upper"]))
        if s["lower"] >= 0:
            buf = torch.empty((p, nx), dtype=torch.float64)
            reqs.append(dist.irecv(buf, s["lower"]))
        for rq in reqs:
            rq.wait()
        if s["lower"] >= 0:
            locg[:p] = buf
        assert torch.equal(locg, ng[zb * p: z1 * p + 1]), "grid shift"
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k3", [(2, 5), (3, 7), (3, 3)])
def test_gloo_exchange_replay(world, k3):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k3, 37, 3, 11, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res

"""Multi-GPU host logic on the CPU (no GPU): the partition plans of
hmg_partition_plan (rank r owns ref-2 blocks [r*320/P, (r+1)*320/P),
i.e. contiguous cells on every level; one-ring halos grouped by owner), checked
against the global mesh, and the halo-exchange protocol run for real between
processes (torch.distributed, gloo, world_size 2) feeding a partitioned
operator apply that must equal the oracle's global apply bit for bit."""
import os
import socket

import numpy as np
import pytest

import hmg_inputs as hi
import oracle

pytest.importorskip("torch")
from paper_1605_00492_b200 import build as hbuild  # noqa: E402

hbuild.build()
from paper_1605_00492_b200 import partition_plan  # noqa: E402


@pytest.fixture(scope="module")
def mesh():
    lam = np.ones((1, 20 * 4 ** 4))
    h = oracle.Hierarchy(4, 2, 1, 0.01, 1e-4, lam)
    yield {r: h.level(r)["nbr"] for r in (2, 3, 4)}
    h.close()


@pytest.mark.parametrize("nranks", [1, 2, 4, 5, 8])
@pytest.mark.parametrize("ref", [2, 3, 4])
def test_plan_matches_global_mesh(mesh, nranks, ref):
    nbr = mesh[ref]
    n = nbr.shape[0]
    plans = [partition_plan(4, ref, r, nranks) for r in range(nranks)]
    owned = np.concatenate([np.arange(p["off"], p["off"] + p["n_own"]) for p in plans])
    assert np.array_equal(owned, np.arange(n))                       # contiguous partition in rank order
    for r, p in enumerate(plans):
        lo, hi_ = p["off"], p["off"] + p["n_own"]
        assert p["off"] == r * n // nranks
        # ownership of every level follows the ref-2 blocks: parents of owned cells are owned one level up
        if ref > 2:
            assert p["off"] % 4 == 0 and p["n_own"] % 4 == 0
        g = nbr[lo:hi_]
        out = np.unique(g[(g < lo) | (g >= hi_)])
        assert np.array_equal(p["halo_gid"], out)                    # halo = out-of-range neighbours, ascending
        loc2glob = np.concatenate([np.arange(lo, hi_), p["halo_gid"]])
        assert np.array_equal(loc2glob[p["nbr_local"]], g)           # local numbering maps back
        # receive runs: consecutive, owner-grouped
        pos = 0
        for q in p["peers"]:
            run = p["halo_gid"][q["recv_offset"]:q["recv_offset"] + q["recv_count"]]
            assert q["recv_offset"] == pos and np.all(run // (n // nranks) == q["rank"])
            pos += q["recv_count"]
        assert pos == len(p["halo_gid"])
    # send lists are exactly the peers' receive runs (same cells, same order)
    for r, p in enumerate(plans):
        for q in p["peers"]:
            peer = plans[q["rank"]]
            back = [x for x in peer["peers"] if x["rank"] == r][0]
            sent = p["off"] + q["send_local"]
            run = peer["halo_gid"][back["recv_offset"]:back["recv_offset"] + back["recv_count"]]
            assert np.array_equal(sent, run)


def _local_apply(L, plan, xloc, nz):
    """Operator apply of the owned rows from local data (R5 order) with the
    bands of the owned global rows."""
    n_own, off = plan["n_own"], plan["off"]
    D, U, H = L["D"][:, off:off + n_own], L["U"][:, off:off + n_own], L["H"][:, :, off:off + n_own]
    Um = np.vstack([np.zeros((1, n_own)), L["U"][:-1, off:off + n_own]])
    nb = plan["nbr_local"]
    y = D * xloc[:, :n_own]
    ks = np.arange(nz)[:, None]
    y = np.where(ks > 0, y + Um * np.vstack([np.zeros((1, n_own)), xloc[:-1, :n_own]]), y)
    y = np.where(ks < nz - 1, y + U * np.vstack([xloc[1:, :n_own], np.zeros((1, n_own))]), y)
    for j in range(3):
        y = y + H[j] * xloc[:, nb[:, j]]
    return y


def test_partitioned_apply_equals_global_single_process():
    """P virtual ranks in one process: owned + halo copies reproduce the global apply bitwise."""
    cfg = hi.Config("part", 4, 2, 8, 0.01, 1e-3)
    lam, b = hi.make_inputs(cfg)
    o = oracle.Hierarchy(4, 2, 8, 0.01, 1e-3, lam)
    for ref in (3, 4):
        L = o.level(ref)
        x = hi.uniform_vector(o.shape(ref), 5 + ref)
        ref_y = o.apply(ref, x)
        for nranks in (2, 4, 8):
            for r in range(nranks):
                p = partition_plan(4, ref, r, nranks)
                xloc = np.concatenate([x[:, p["off"]:p["off"] + p["n_own"]], x[:, p["halo_gid"]]], axis=1)
                y = _local_apply(L, p, xloc, 8)
                assert np.array_equal(y, ref_y[:, p["off"]:p["off"] + p["n_own"]])
    o.close()


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = hi.Config("part", 4, 2, 8, 0.01, 1e-3)
    lam, b = hi.make_inputs(cfg)
    o = oracle.Hierarchy(4, 2, 8, 0.01, 1e-3, lam)
    ok = True
    nz = 8
    for ref in (3, 4):
        L = o.level(ref)
        x = hi.uniform_vector(o.shape(ref), 11 + ref)
        p = partition_plan(4, ref, rank, world)
        n_own = p["n_own"]
        own = x[:, p["off"]:p["off"] + n_own]
        # the exchange protocol of halo_exchange(): per peer a cell-major
        # [cells][nz] buffer of my owned cells it needs; receive into my halo run
        xloc = np.zeros((nz, n_own + len(p["halo_gid"])))
        xloc[:, :n_own] = own
        reqs, recvs = [], []
        for q in p["peers"]:
            send = torch.from_numpy(np.ascontiguousarray(own[:, q["send_local"]].T))
            recv = torch.empty((q["recv_count"], nz), dtype=torch.float64)
            reqs.append(dist.isend(send, q["rank"]))
            reqs.append(dist.irecv(recv, q["rank"]))
            recvs.append((q, recv))
        for rq in reqs:
            rq.wait()
        for q, recv in recvs:
            xloc[:, n_own + q["recv_offset"]:n_own + q["recv_offset"] + q["recv_count"]] = recv.numpy().T
        y = _local_apply(L, p, xloc, nz)
        ok = ok and np.array_equal(y, o.apply(ref, x)[:, p["off"]:p["off"] + n_own])
        # distributed inner product: all-reduce of rank-local sums
        t = torch.tensor([float(np.sum(own * own))], dtype=torch.float64)
        dist.all_reduce(t)
        ok = ok and abs(t.item() - float(np.sum(x * x))) <= 1e-12 * float(np.sum(x * x))
    o.close()
    with open(f"{result_path}.{rank}", "w") as fh:
        fh.write("ok" if ok else "FAIL")
    dist.destroy_process_group()


def test_halo_exchange_gloo_world_size_2(tmp_path):
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    res = str(tmp_path / "res")
    mp.spawn(_worker, args=(2, port, res), nprocs=2, join=True)
    for r in range(2):
        assert open(f"{res}.{r}").read() == "ok"

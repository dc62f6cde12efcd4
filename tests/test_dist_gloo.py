"""Multi-rank host logic on CPU (gloo, world sizes 2 and 3): row partition, halo plan, halo
exchange into the extended arrays, all-reduce of the partial sums.  The oracle stands in for the
kernels on each rank's local CSR; the sharded results must equal the single-process oracle."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, n, k, p, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, name, n, k, p, q)
    except Exception as e:  # report instead of leaving the parent waiting on the queue
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, world, name, n, k, p, q):
    if True:
        import oracle
        from paper_2605_26975_b200 import plp
        from paper_2605_26975_b200.dist import HaloPlan, HaloExchange
        from plp_inputs import make_config, permute_graph, draw_U, draw_eta
        g0 = make_config(name, n=n)
        g = permute_graph(g0, plp.tile_order(g0.row_ptr, g0.col))
        U = draw_U(g.n, k, 5)
        eta = draw_eta(g.n, k, 5)
        plan = HaloPlan(g.row_ptr, g.col, g.w, rank, world, k)
        plan.exchange_lists()

        def pack(idx, X, out):
            out.copy_(X.index_select(0, idx))

        xchg = HaloExchange(plan, k, "cpu", pack=pack)
        U_ext = torch.zeros(plan.n_loc + plan.n_halo, k, dtype=torch.float64)
        E_ext = torch.zeros_like(U_ext)
        U_ext[:plan.n_loc] = torch.from_numpy(U[plan.r0:plan.r1])
        E_ext[:plan.n_loc] = torch.from_numpy(eta[plan.r0:plan.r1])
        xchg(U_ext)
        xchg(E_ext)
        ok_halo = np.array_equal(U_ext[plan.n_loc:].numpy(), U[plan.halo]) and \
            np.array_equal(E_ext[plan.n_loc:].numpy(), eta[plan.halo])

        class Loc:
            row_ptr, col, w = plan.rp_loc, plan.col_loc, plan.w_loc

        Ue, Ee = U_ext.numpy(), E_ext.numpy()
        AB = torch.from_numpy(np.concatenate([oracle.numerators(Loc, Ue, p),
                                              oracle.pnorms(Ue, p, n_rows=plan.n_loc)]))
        dist.all_reduce(AB)
        A, B = AB[:k].numpy(), AB[k:].numpy()
        G = oracle.euc_grad(Loc, Ue, p, A, B)
        Hv = oracle.hessvec(Loc, Ue, Ee, p, 1e-9, "sparse", (A, B))
        F, A0, B0, G0, H0 = oracle.fgrad_hessvec(g, U, eta, p)
        sl = slice(plan.r0, plan.r1)

        def rel(x, r):
            return float(np.max(np.abs(x - r)) / max(np.max(np.abs(r)), 1e-300))

        q.put((rank, ok_halo, rel(A, A0), rel(B, B0), rel(G, G0[sl]), rel(Hv, H0[sl]),
               plan.n_loc, plan.n_halo, int((plan.recv_cnt > 0).sum()), int((plan.send_cnt > 0).sum())))


@pytest.mark.parametrize("name,n,k,p,world", [("C1", 600, 3, 1.5, 2), ("C5", 6000, 8, 1.2, 2),
                                               ("C5", 6000, 4, 1.37, 3)])
def test_sharded_oracle_matches_single(name, n, k, p, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n, k, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    errs = [r for r in res if r[1] == "error"]
    assert not errs, errs
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert sum(r[6] for r in res) == n if name != "C1" else True
    for (rank, ok_halo, eA, eB, eG, eH, n_loc, n_halo, n_recv, n_send) in res:
        assert ok_halo, f"rank {rank}: halo rows differ after the exchange"
        assert eA < 1e-13 and eB < 1e-13, (eA, eB)
        assert eG < 1e-12 and eH < 1e-12, (eG, eH)
        assert n_halo > 0 and n_recv >= 1 and n_send >= 1

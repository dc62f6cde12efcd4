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


# ---- the collective k-means protocol (plp_kmeans_dist, csrc/kmeans.cu) on CPU ranks --------------
# Each rank holds a contiguous block of the points; the local steps are plain numpy (a stand-in for
# the kernels), the cross-rank steps are the protocol's all-reduces: row counts, per-rank D^2 sums
# (the rank whose running sum crosses u * sum picks inside its block and broadcasts the point),
# per-cluster sums / counts / sse, and the farthest point (value, global index) for an empty
# cluster.  The result must be the sequential k-means of the oracle on the concatenated points.
def _kmeans_protocol(X, K, u_all, restarts, max_iters=300, rel_tol=1e-9):
    rank, world = dist.get_rank(), dist.get_world_size()
    n, dim = X.shape
    cnt = torch.zeros(world, dtype=torch.float64)
    cnt[rank] = n
    dist.all_reduce(cnt)
    off = np.concatenate([[0], np.cumsum(cnt.numpy().astype(np.int64))])
    N, my0 = int(off[-1]), int(off[rank])

    def bcast(row_or_none):
        v = torch.zeros(dim, dtype=torch.float64)
        if row_or_none is not None:
            v += torch.from_numpy(row_or_none)
        dist.all_reduce(v)
        return v.numpy()

    def mine(gi):
        return X[gi - my0] if my0 <= gi < my0 + n else None

    best = (np.inf, None, None, 0)
    u_all = np.asarray(u_all, dtype=np.float64).reshape(-1)
    for r in range(restarts):
        u = u_all[r * K:(r + 1) * K]
        C = np.zeros((K, dim))
        c0 = min(int(np.floor(u[0] * N)), N - 1)
        C[0] = bcast(mine(c0))
        D2 = None
        for m in range(1, K):
            d = ((X - C[m - 1]) ** 2).sum(axis=1)
            D2 = d if D2 is None else np.minimum(D2, d)
            S_r = torch.zeros(world, dtype=torch.float64)
            S_r[rank] = D2.sum()
            dist.all_reduce(S_r)
            S_r = S_r.numpy()
            S = float(S_r.sum())
            row = None
            if not S > 0.0:
                row = mine(min(int(np.floor(u[m] * N)), N - 1))
            else:
                t = u[m] * S
                pre = np.concatenate([[0.0], np.cumsum(S_r)])
                own = next((q for q in range(world) if pre[q] <= t < pre[q + 1]),
                           max(q for q in range(world) if S_r[q] > 0))
                if own == rank:
                    cs = np.cumsum(D2)
                    hit = np.nonzero(cs > t - pre[own])[0]
                    row = X[hit[0] if hit.size else int(np.max(np.nonzero(D2 > 0)[0]))]
            C[m] = bcast(row)

        def assign(C):
            dd = ((X[:, None, :] - C[None, :, :]) ** 2).sum(axis=2)
            lab = np.argmin(dd, axis=1)
            bd = dd[np.arange(n), lab]
            red = np.zeros(K * dim + K + 1)
            for c in range(K):
                red[c * dim:(c + 1) * dim] = X[lab == c].sum(axis=0)
                red[K * dim + c] = np.sum(lab == c)
            red[-1] = bd.sum()
            red = torch.from_numpy(red)
            dist.all_reduce(red)
            return lab, bd, red.numpy()

        lab, bd, red = assign(C)
        cur, it = red[-1], 0
        while it < max_iters:
            for c in range(K):
                if red[K * dim + c] > 0:
                    C[c] = red[c * dim:(c + 1) * dim] / red[K * dim + c]
            for c in range(K):
                if red[K * dim + c] > 0:
                    continue
                vi = torch.zeros(2 * world, dtype=torch.float64)
                if n:
                    j = int(np.argmax(bd))
                    vi[2 * rank], vi[2 * rank + 1] = bd[j], my0 + j
                dist.all_reduce(vi)
                vi = vi.numpy()
                own = max(range(world), key=lambda q: (vi[2 * q], -q))
                row = None
                if own == rank:
                    j = int(vi[2 * own + 1]) - my0
                    row, bd[j] = X[j].copy(), -1.0
                C[c] = bcast(row)
            lab, bd, red = assign(C)
            it += 1
            nxt = red[-1]
            conv = cur == 0.0 or abs(cur - nxt) < rel_tol * cur
            cur = nxt
            if conv:
                break
        if cur < best[0]:
            best = (cur, lab.copy(), C.copy(), it)
    return best


def _km_worker(rank, world, port, n, dim, K, seed, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from plp_inputs import draw_uniforms
        rng = np.random.default_rng(seed)
        X = rng.uniform(-8, 8, size=(K, dim))[rng.integers(0, K, n)] + rng.standard_normal((n, dim))
        if seed % 2:  # duplicates: empty clusters and the farthest-point reseed
            X[: n // 2] = X[0]
        u = draw_uniforms(3, K)
        b = np.linspace(0, n, world + 1).astype(int)
        b[1] = b[1] // 3  # unequal blocks
        sse, lab, C, it = _kmeans_protocol(X[b[rank]:b[rank + 1]], K, u, restarts=3)
        lab_o, C_o, sse_o, it_o = oracle.kmeans(X, K, u, restarts=3)
        q.put((rank, bool(np.array_equal(lab, lab_o[b[rank]:b[rank + 1]])),
               float(np.max(np.abs(C - C_o)) / np.max(np.abs(C_o))), abs(sse - sse_o) / sse_o, it == it_o))
    except Exception as e:
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,dim,K,seed,world", [(3000, 4, 5, 0, 2), (2500, 8, 8, 1, 3), (4001, 3, 3, 2, 3)])
def test_kmeans_collective_protocol_matches_oracle(n, dim, K, seed, world):
    """The protocol of plp_kmeans_dist on 2 and 3 gloo ranks (unequal row blocks, empty clusters)
    gives the oracle's sequential k-means: labels equal, centroids and sse within 1e-12."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_km_worker, args=(r, world, port, n, dim, K, seed, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    errs = [r for r in res if r[1] == "error"]
    assert not errs, errs
    for rank, same_lab, eC, eS, same_it in res:
        assert same_lab, f"rank {rank}: labels differ"
        assert eC < 1e-12 and eS < 1e-12, (eC, eS)
        assert same_it

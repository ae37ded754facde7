"""Multi-process CPU run of the C++ distributed driver over torch.distributed
(gloo): world sizes 2 (1x2 grid) and 4 (2x2 grid), one process per rank, the
driver's collectives routed through qdwhg_comm_callbacks-style callbacks
(broadcasts / all-reductions on the grid's row and column sub-groups, grouped
point-to-point exchanges).  Local compute is the host test engine
(tests/cpp/dist_host.cpp); rank 0's result is checked against the oracle."""
import ctypes
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "cpp", "libqdwhg_disthost.so")

CB_BCAST = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                            ctypes.c_int)
CB_ALLRED = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                             ctypes.c_int)
CB_SEND = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int)
CB_GROUP = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)


class Callbacks(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("bcast", CB_BCAST), ("allreduce", CB_ALLRED), ("send", CB_SEND),
                ("recv", CB_SEND), ("group_begin", CB_GROUP), ("group_end", CB_GROUP)]


def rank_main(rank, world, P, Q, port, out_path):
    """One process: gloo init, grid sub-groups, callbacks, the driver."""
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from oracle import qdwh_oracle as O
    from paper_2104_14186_b200 import matgen
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    rows = [dist.new_group([p * Q + q for q in range(Q)]) for p in range(P)]
    cols = [dist.new_group([p * Q + q for p in range(P)]) for q in range(Q)]
    me_p, me_q = rank // Q, rank % Q
    groups = {0: None, 1: rows[me_p], 2: cols[me_q]}
    ops = {0: dist.ReduceOp.SUM, 1: dist.ReduceOp.MAX, 2: dist.ReduceOp.MIN}
    state = {"depth": 0, "p2p": []}

    def arr(buf, count):
        return torch.from_numpy(np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ctypes.c_double)),
                                                      shape=(count,)))

    def bcast(ctx, buf, count, root, team):
        if count:
            dist.broadcast(arr(buf, count), src=root, group=groups[team])
        return 0

    def allreduce(ctx, buf, count, op, team):
        if count:
            dist.all_reduce(arr(buf, count), op=ops[op], group=groups[team])
        return 0

    def p2p(kind):
        def f(ctx, buf, count, peer):
            op = dist.P2POp(dist.isend if kind == "send" else dist.irecv, arr(buf, count), peer)
            state["p2p"].append(op)
            if state["depth"] == 0:
                flush()
            return 0
        return f

    def flush():
        if state["p2p"]:
            for req in dist.batch_isend_irecv(state["p2p"]):
                req.wait()
            state["p2p"] = []

    def gbegin(ctx):
        state["depth"] += 1
        return 0

    def gend(ctx):
        state["depth"] -= 1
        if state["depth"] == 0:
            flush()
        return 0

    cbs = Callbacks(None, CB_BCAST(bcast), CB_ALLRED(allreduce), CB_SEND(p2p("send")), CB_SEND(p2p("recv")),
                    CB_GROUP(gbegin), CB_GROUP(gend))
    lib = ctypes.CDLL(LIB)
    P_, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    lib.dh_partial_eig_rank.argtypes = [I, I, I, I, P_, I64, P_, I64, D, I64, P_, P_, I64, P_, P_, P_, P_, I]
    n, nb, k = 160, 32, 16
    lam = matgen.config_eigenvalues("uniform", n, 42)
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, 42))
    a = np.asfortranarray(0.5 * ((q * lam) @ q.T + ((q * lam) @ q.T).T))
    c = matgen.largest_k_shift(lam, k)
    vals = np.zeros(n)
    V = np.zeros((n, n), order="F")
    ko, ello, mu = I64(0), I64(0), D(0)
    err = ctypes.create_string_buffer(512)
    rc = lib.dh_partial_eig_rank(P, Q, nb, rank, ctypes.byref(cbs), n, a.ctypes.data, n, c, k,
                                 vals.ctypes.data, V.ctypes.data, n, ctypes.byref(ko), ctypes.byref(ello),
                                 ctypes.byref(mu), err, 512)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    np.savez(out_path % rank, vals=vals[:ko.value], v=V[:, :ko.value], ell=ello.value, mu=mu.value, a=a, c=c,
             k=k)
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("P,Q", [(1, 2), (2, 2)])
def test_gloo_multiprocess_partial_eig(tmp_path, P, Q):
    from oracle import qdwh_oracle as O
    subprocess.check_call(["make", "-s", "-C", os.path.join(HERE, "cpp")])
    world = P * Q
    port = free_port()
    out = str(tmp_path / "rank%d.npz")
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r); import test_dist_gloo as t; "
            "t.rank_main(int(sys.argv[1]), %d, %d, %d, %d, %r)" % (ROOT, HERE, world, P, Q, port, out))
    procs = [subprocess.Popen([sys.executable, "-c", code, str(r)], cwd=ROOT, env=dict(os.environ, OMP_NUM_THREADS="1"))
             for r in range(world)]
    rcs = [p.wait(timeout=300) for p in procs]
    assert rcs == [0] * world, rcs
    res = [np.load(out % r) for r in range(world)]
    r0 = res[0]
    a, c, k = r0["a"], float(r0["c"]), int(r0["k"])
    ref = O.qdwh_partial_eig(c * np.eye(a.shape[0]) - a, O.choose_shift(3))
    assert len(r0["vals"]) == k == ref.count()
    np.testing.assert_allclose(r0["vals"], c - ref.lambda_minus[:k], rtol=1e-10)
    assert int(r0["ell"]) == ref.subspace_size
    for r in res[1:]:  # every rank agrees on the values
        np.testing.assert_array_equal(r["vals"], r0["vals"])
    v = r0["v"]
    n = a.shape[0]
    assert np.linalg.norm(a @ v - v * r0["vals"]) / np.linalg.norm(a) <= 1e-12 * np.sqrt(n)
    assert np.linalg.norm(np.eye(k) - v.T @ v) <= 1e-12 * np.sqrt(n)

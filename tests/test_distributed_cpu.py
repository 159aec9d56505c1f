"""N > 1 host path on CPU: world_size 2 and 4 over torch.distributed gloo.

Every rank builds the Low-NN partition and its comm plan with libesg_b200's
host code, then runs the forward block by block (oracle numerics) with a
halo exchange before each of the 2*M blocks that follows exactly the routing
the CUDA library issues through NCCL (pack send rows per neighbour, one
send/recv per neighbour, receive straight into the contiguous halo rows).
The gathered outputs must equal the serial forward bit for bit
(test_runtime.cpp:235-271; acceptance.cpp:244-355 exchange counting)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2507_03840_b200 import esg

BASIS = {72: [0, 1], 8: [0, 1]}


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def problem():
    s = esg.make_jittered_lattice(120, 2.2, 0.45, [72, 8, 8], 3)
    g = O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), 4.5)
    return s, g


def halo_exchange(nodes, plan, counter):
    """One exchange: pack send rows per peer, isend all, recv into halo rows."""
    reqs = []
    at = 0
    bufs = []
    for q, peer in enumerate(plan["nbr_peer"]):
        n = plan["nbr_send_count"][q]
        rows = plan["send_rows"][at:at + n]
        at += n
        buf = torch.from_numpy(np.ascontiguousarray(nodes[rows]))
        bufs.append(buf)
        reqs.append(dist.isend(buf, int(peer)))
    for q, peer in enumerate(plan["nbr_peer"]):
        r0, n = plan["nbr_recv_row"][q], plan["nbr_recv_count"][q]
        buf = torch.empty((n,) + nodes.shape[1:], dtype=torch.from_numpy(nodes[:1]).dtype)
        dist.recv(buf, int(peer))
        nodes[r0:r0 + n] = buf.numpy()
    for r in reqs:
        r.wait()
    counter[0] += 1
    counter[1] += len(plan["nbr_peer"])


def worker(rank, world, port, dtype, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, g = problem()
        deg = O.in_degrees(s.n_atoms, g)
        depth = int(np.log2(world))
        part = esg.lownn_partition(s, deg, depth, 4.5)
        off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        plan = esg.CommPlan(None, s.species, part, world, rank, csr=(off, g["src"])).export()
        plan["n_rows"] = len(plan["row_global"])
        plan["n_owned"] = int(np.sum(part == rank))
        view = O.plan_view(plan, s.species, g)
        m = O.Model(2, 8, 2, 8, 4.5, 1, BASIS)
        nodes, edges = m.init_tables(view, dtype)
        counter = [0, 0]
        for layer in range(2):
            for nb in (True, False):
                halo_exchange(nodes, plan, counter)
                m.block(view, nodes, edges, layer, nb)
        no, eo = m.heads(view, nodes, edges)
        q.put((rank, plan["row_global"][:plan["n_owned"]], plan["edge_index"], no, eo, counter,
               len(plan["nbr_peer"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_distributed_forward_matches_serial_bitwise(world, dtype):
    s, g = problem()
    m = O.Model(2, 8, 2, 8, 4.5, 1, BASIS)
    sno, seo = m.forward(O.serial_view(s.n_atoms, s.species, g), dtype)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, dtype, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    no = np.zeros_like(sno)
    eo = np.zeros_like(seo)
    seen = np.zeros(len(seo), bool)
    for rank, owned, eidx, rno, reo, counter, n_nb in res:
        no[owned] = rno
        eo[eidx] = reo
        seen[eidx] = True
        # exactly 2*M exchanges, one message per neighbour per exchange
        assert counter[0] == 4 and counter[1] == 4 * n_nb
    assert seen.all()
    assert np.array_equal(no, sno) and np.array_equal(eo, seo)


# ---------------------------------------------------------------- training
def halo_backward(g_nodes, plan):
    """Reverse of halo_exchange (distributed.h:98-129): send halo-row
    gradients back to their owners, add them into the send rows in
    ascending peer order, then zero the halo rows."""
    reqs, bufs = [], []
    for q, peer in enumerate(plan["nbr_peer"]):
        r0, n = plan["nbr_recv_row"][q], plan["nbr_recv_count"][q]
        buf = torch.from_numpy(np.ascontiguousarray(g_nodes[r0:r0 + n]))
        bufs.append(buf)
        reqs.append(dist.isend(buf, int(peer)))
    at = 0
    for q, peer in enumerate(plan["nbr_peer"]):
        n = plan["nbr_send_count"][q]
        rows = plan["send_rows"][at:at + n]
        at += n
        buf = torch.empty((n,) + g_nodes.shape[1:], dtype=torch.from_numpy(g_nodes[:1]).dtype)
        dist.recv(buf, int(peer))
        g_nodes[rows] += buf.numpy()
    for r in reqs:
        r.wait()
    for q in range(len(plan["nbr_peer"])):
        r0, n = plan["nbr_recv_row"][q], plan["nbr_recv_count"][q]
        g_nodes[r0:r0 + n] = 0


def train_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, g = problem()
        deg = O.in_degrees(s.n_atoms, g)
        part = esg.lownn_partition(s, deg, int(np.log2(world)), 4.5)
        off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        plan = esg.CommPlan(None, s.species, part, world, rank, csr=(off, g["src"])).export()
        plan["n_rows"] = len(plan["row_global"])
        plan["n_owned"] = int(np.sum(part == rank))
        view = O.plan_view(plan, s.species, g)
        m = O.Model(2, 8, 2, 8, 4.5, 1, BASIS)
        nt, nm, et, em, nt64, et64 = m.toy_targets(s.n_atoms, s.species, g)
        owned = plan["row_global"][:plan["n_owned"]]
        ei = plan["edge_index"]
        targets = (nt64[owned], nm[owned], et64[ei], em[ei])
        local = int(nm[owned].sum() + em[ei].sum())
        cnt = torch.tensor([float(local)], dtype=torch.float64)
        allc = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allc, cnt)  # allreduce_count
        n_total = int(sum(float(c) for c in allc))
        counter = [0, 0]
        (sa, sq, c), grads = O.loss_grad(m, view, targets, n_total, np.float64,
                                         exchange=lambda nodes: halo_exchange(nodes, plan, counter),
                                         exchange_bwd=lambda gn: halo_backward(gn, plan))
        mine = torch.from_numpy(np.concatenate([grads, [sa, sq, c]]))
        alls = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(alls, mine)  # allreduce_gradients: rank order, fp64
        tot = np.zeros_like(mine.numpy())
        for p in range(world):
            tot = tot + alls[p].numpy()
        q.put((rank, n_total, tot))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_training_step_matches_serial(world):
    """test_runtime.cpp:330-388: the distributed loss and rank-summed
    gradients equal the serial step (fp64, <= 1e-10)."""
    s, g = problem()
    m = O.Model(2, 8, 2, 8, 4.5, 1, BASIS)
    nt, nm, et, em, nt64, et64 = m.toy_targets(s.n_atoms, s.species, g)
    n_total = int(nm.sum() + em.sum())
    (sa, sq, _), sgrads = O.loss_grad(m, O.serial_view(s.n_atoms, s.species, g), (nt64, nm, et64, em), n_total,
                                      np.float64)
    sloss = (sa + sq) / n_total
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=train_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, total, tot in res:
        assert total == n_total
        loss = (tot[-3] + tot[-2]) / total
        assert abs(loss - sloss) <= 1e-12 * abs(sloss)
        gr = tot[:-3]
        assert np.abs(gr - sgrads).max() <= 1e-10 * max(1.0, np.abs(sgrads).max())
    # replicas land on identical sums
    assert all(np.array_equal(res[0][2], r[2]) for r in res)

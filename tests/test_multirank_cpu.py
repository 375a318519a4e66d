"""World-size-2 CPU tests (gloo) of the host-side logic of the expert-parallel (N > 1) path:
the NCCL unique-id broadcast used to build the communicator, and the exchange plan
(lancet_plan_exchange) from which every grouped NCCL send/recv is posted -- including the
pairwise matching condition NCCL requires (the k-th send from rank a to rank b has the size
of the k-th receive b posts from a)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, tmpdir, case):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        globals()[case](rank, world)
        open(os.path.join(tmpdir, f"ok{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


def _spawn(case, world=2):
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_run, args=(world, _free_port(), tmp, case), nprocs=world, join=True)
        assert all(os.path.exists(os.path.join(tmp, f"ok{r}")) for r in range(world))


def case_nccl_id(rank, world):
    from paper_2404_19429_b200 import lancet
    nid = lancet.share_nccl_id(None, rank)
    ids = [None] * world
    dist.all_gather_object(ids, nid)
    assert len(nid) == 128 and all(i == ids[0] for i in ids)


def _posted(plan, G, E_l, n, rank, send, recv, serial=False):
    """The (peer -> list of bytes) sends and receives the scheduler posts for one dispatch
    all-to-all per chunk (stage order), mirroring lancet.cu."""
    sends = {p: [] for p in range(G)}
    recvs = {p: [] for p in range(G)}
    chunks = [list(range(n))] if serial else [[c] for c in range(n)]
    for cs in chunks:
        for p in range(G):
            for i in range(E_l):
                e = p * E_l + i
                for c in cs:
                    sends[p].append(int(send[e, c]))
        for p in range(G):
            for el in range(E_l):
                for c in cs:
                    recvs[p].append(int(recv[p, el, c]))
    return sends, recvs


def case_exchange_plan(rank, world):
    import synthetic as S
    from oracle import moe
    from paper_2404_19429_b200 import lancet
    E_l, n, k = 2, 3, 2
    E = world * E_l
    T = 300 + 57 * rank                                   # T may differ per rank
    sh = S.LayerShape(T=T, d=32, f=64, E=E, G=world, k=k, cf=1.0, n_chunks=n)
    ins = S.gen_rank_inputs(11, rank, sh, beta=1.0)
    rt = moe.route_rank(ins["x"], ins["wg"], k, 1.0, n)
    send = rt.counts.astype(np.int32)                      # [E][n]
    # the size all-to-all: every rank learns what each source sends to its experts
    sends = [None] * world
    dist.all_gather_object(sends, send)
    recv = moe.recv_counts(sends, world, rank).astype(np.int32)   # [G][E_l][n]
    plan = lancet.plan_exchange(world, E_l, n, send, recv)

    # send side: S is the chunk prefix, experts packed 128-row aligned, chunks contiguous
    assert np.array_equal(plan["S"][:, 1:] - plan["S"][:, :-1], send)
    ends = plan["send_off"] + plan["S"][:, -1]
    assert np.all(plan["send_off"] % 128 == 0)
    assert np.all(plan["send_off"][1:] >= ends[:-1])
    # receive side: groups (chunk, local expert) hold the sum over sources, 128-aligned,
    # expert-major in memory, rows ordered by source inside a group
    assert np.array_equal(plan["grp_rows"], recv.sum(0).T)
    offs = [(int(plan["grp_off"][c, el]), int(plan["grp_rows"][c, el]))
            for el in range(E_l) for c in range(n)]
    assert all(o % 128 == 0 for o, _ in offs)
    for (o0, r0), (o1, _) in zip(offs, offs[1:]):
        assert o1 == o0 + -(-r0 // 128) * 128
    assert plan["total_rows"] == offs[-1][0] + -(-offs[-1][1] // 128) * 128
    assert np.array_equal(plan["src_off"], np.cumsum(recv, axis=0) - recv)

    # NCCL matching: rank a's k-th send to b has the size of b's k-th receive from a
    mine = {}
    for serial in (False, True):
        mine[serial] = _posted(plan, world, E_l, n, rank, send, recv, serial)
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    for serial in (False, True):
        for a in range(world):
            for b in range(world):
                assert allp[a][serial][0][b] == allp[b][serial][1][a], (serial, a, b)


def test_nccl_unique_id_broadcast_over_gloo():
    _spawn("case_nccl_id")


def test_exchange_plan_two_ranks_over_gloo():
    _spawn("case_exchange_plan")


def test_plan_rejects_bad_arguments():
    from paper_2404_19429_b200 import lancet
    with pytest.raises(lancet.LancetError):
        lancet.plan_exchange(2, 1, 1, np.array([[1], [-1]]), np.zeros((2, 1, 1)))

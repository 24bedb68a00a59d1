"""world_size-2 gloo test of the multi-rank host logic on CPU: every rank
builds the same schedule through the C ABI, the per-rank parameter layouts
partition the LLM exactly once and replicate the DP modules, and the
max-over-ranks timing reduction used by bench.py agrees on all ranks."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import ctypes as C
        from synth import get_config, param_specs
        from paper_2605_25451_b200 import _lib as L
        from paper_2605_25451_b200 import schedule as BS
        from paper_2605_25451_b200.runtime import model_cfg
        cfg = get_config("C1", P=world, M=4, V=1)
        sched = BS.build(world, 4, 1)
        text = sched.serialize()
        mc = model_cfg(cfg, "bf16")
        sc = BS.make_cfg(world, 4, 1)
        n, tot, dp = C.c_int32(), C.c_int64(), C.c_int64()
        L.call("bm_param_count", C.byref(mc), C.byref(sc), rank, C.byref(n), C.byref(tot), C.byref(dp))
        names = []
        for i in range(n.value):
            pi = L.ParamInfo()
            L.call("bm_param_info_get", C.byref(mc), C.byref(sc), rank, i, C.byref(pi))
            names.append((pi.name.decode(), pi.kind))
        gathered = [None] * world
        dist.all_gather_object(gathered, (text, names))
        ok = all(g[0] == text for g in gathered)
        llm = [nm for g in gathered for nm, k in g[1] if k == 1]
        dpn = [set(nm for nm, k in g[1] if k == 0) for g in gathered]
        all_llm = {nm for nm, _, _ in param_specs(cfg) if nm.startswith("llm.")}
        ok &= sorted(llm) == sorted(all_llm) and len(llm) == len(set(llm))
        ok &= all(d == dpn[0] for d in dpn)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok &= t.item() == world
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, bool(ok), ""))
    except Exception as e:  # pragma: no cover
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("world", [2, 4])
def test_multirank_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


def _replica_worker(rank, world, P, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2605_25451_b200.runtime import exchange
        cnt = [0]

        def new_id():
            cnt[0] += 1
            return f"id-{rank}-{cnt[0]}".encode()
        peers, ids, allp = exchange(None, P, world // P, rank, f"ipc-{rank}", new_id)
        assert allp == [f"ipc-{g}" for g in range(world)], allp
        got = [None] * world
        dist.all_gather_object(got, (peers, ids))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, got, ""))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, repr(e)))


@pytest.mark.parametrize("world,P", [(4, 2), (2, 1), (4, 4), (8, 4)])
def test_replica_exchange_groups(world, P):
    """D = world / P pipeline replicas: IPC peers are the process's own replica
    (stage order), every process of a replica shares one pipeline id, every
    process the world id, and the D processes of a stage one stage id -- each id
    distinct per group."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, world, P, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(g is not None for _, g, _ in res), res
    got = res[0][1]
    D = world // P
    for r, (peers, ids) in enumerate(got):
        rep, st = divmod(r, P)
        assert peers == [f"ipc-{rep * P + s}" for s in range(P)]
        assert ids["pipe"] == (got[rep * P][1]["pipe"] if P > 1 else None)
        assert ids["world"] == (b"id-0-" + (b"2" if P > 1 else b"1") if D > 1 else None)
        assert ids["stage"] == (got[st][1]["stage"] if D > 1 else None)
    if P > 1:
        assert len({got[k * P][1]["pipe"] for k in range(D)}) == D
    if D > 1:
        assert len({got[s][1]["stage"] for s in range(P)}) == P


def test_sum_mode_selection(monkeypatch):
    """Step-end sums: NCCL when every process owns a GPU, the library's peer-memory
    sum when two processes share one (NCCL rejects duplicate devices), forced by
    BM_STEP_SUM."""
    from paper_2605_25451_b200.runtime import sum_mode
    monkeypatch.delenv("BM_STEP_SUM", raising=False)
    assert sum_mode(["a", "b", "c", "d"]) == "nccl"
    assert sum_mode(["a", "a"]) == "peer"
    assert sum_mode(["a", "b", "a", "b"]) == "peer"
    monkeypatch.setenv("BM_STEP_SUM", "peer")
    assert sum_mode(["a", "b"]) == "peer"
    monkeypatch.setenv("BM_STEP_SUM", "nccl")
    assert sum_mode(["a", "a"]) == "nccl"

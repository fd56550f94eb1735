"""Multi-GPU host logic on CPU (single process and gloo world_size 2), and the row-panel
per-rank code on one GPU with virtual ranks (-m gpu)."""
import os
import socket

import numpy as np
import pytest

import synth
from oracle import chain, tables


def _upper_codes(n):
    nt = (n + 255) // 256
    return {(I << 16) | J for I in range(nt) for J in range(I, nt)}


@pytest.mark.parametrize("n,P", [(256, 1), (1024, 2), (4096, 3), (4096, 8), (16384, 8), (16384, 5)])
def test_rowpanel_tiles_partition(n, P):
    """Every upper 256-tile is computed by exactly one rank; loads differ by at most one tile."""
    from paper_2507_09165_b200 import dist
    seen, counts = [], []
    for r in range(P):
        codes, real = dist.rowpanel_tiles(n, P, r)
        assert len(codes) == len(dist.rowpanel_tiles(n, P, 0)[0])          # equal packed size
        assert all(c == 0xFFFFFFFF for c in codes[real:])
        seen += codes[:real]
        counts.append(real)
    assert len(seen) == len(set(seen)) and set(seen) == _upper_codes(n)
    assert max(counts) - min(counts) <= 1


def test_shard_range_covers_batch():
    from paper_2507_09165_b200 import dist
    for B in [1, 7, 32, 33]:
        for W in [1, 2, 4, 8]:
            got = []
            for r in range(W):
                f, c = dist.shard_range(B, W, r)
                got += list(range(f, f + c))
            assert got == list(range(B))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_09165_b200 import dist
        # (1) each rank's tile list, gathered: a disjoint cover of the upper tiles
        codes, real = dist.rowpanel_tiles(4096, world, rank)
        t = torch.tensor(codes, dtype=torch.int64)
        allc = [torch.zeros_like(t) for _ in range(world)]
        tdist.all_gather(allc, t)
        flat = [int(v) for a in allc for v in a.tolist() if int(v) != 0xFFFFFFFF]
        ok_tiles = len(flat) == len(set(flat)) == 136
        # (2) batch shards of config c4 gathered: the global batch exactly once
        f, c = dist.shard_range(32, world, rank)
        r = torch.tensor([f, c], dtype=torch.int64)
        allr = [torch.zeros_like(r) for _ in range(world)]
        tdist.all_gather(allr, r)
        idx = sorted(i for a in allr for i in range(int(a[0]), int(a[0]) + int(a[1])))
        # (3) the NCCL unique id broadcast over the process group: identical bytes on every rank
        try:
            uid = dist.broadcast_nccl_id()
            u = torch.tensor(list(uid[:16]), dtype=torch.int64)
            allu = [torch.zeros_like(u) for _ in range(world)]
            tdist.all_gather(allu, u)
            ok_uid = all(torch.equal(allu[0], a) for a in allu) and any(uid)
        except Exception as exc:   # libnccl.so.2 not loadable on this host
            ok_uid = "skip: %s" % exc
        q.put((rank, ok_tiles, idx == list(range(32)), ok_uid))
    finally:
        tdist.destroy_process_group()


def test_gloo_world2_host_logic():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_tiles, ok_shard, ok_uid in res:
        assert ok_tiles and ok_shard
        assert ok_uid is True or str(ok_uid).startswith("skip")


# ---------------------------------------------------------------- GPU: virtual ranks

@pytest.mark.gpu
@pytest.mark.parametrize("n,P,prec", [(512, 2, "fp16"), (768, 3, "fp16"), (1024, 4, "tf32"), (2048, 8, "fp16"),
                                      (1024, 1, "bf16")])
def test_rowpanel_virtual_parity(n, P, prec):
    """The row-panel per-rank code (tiles per rank, packed outputs, gather order, unpack with
    mirror) with P virtual ranks on one GPU, vs the oracle; output exactly symmetric."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2507_09165_b200 as pkg
    X = synth.goe(n, synth.SEED_BASE + n + P)
    f = pkg.Filter(pkg.filters.half_filter(), precision=prec)
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    P_gpu = f.project_rowpanel_virtual(Xd, P).double().cpu().numpy()
    assert f.status() == "PSD_OK"
    lam = chain.frobenius_bound(X)
    ref, _ = chain.project(X, tables.F_HALF_REFINED, tables.half_kappas(7), lam=lam)
    err = np.linalg.norm(P_gpu - ref) / np.linalg.norm(ref)
    assert err <= {"fp16": 5e-3, "tf32": 5e-3, "bf16": 3e-2}[prec], err
    assert np.array_equal(P_gpu, P_gpu.T)
    # and the sign output
    S = f.project_rowpanel_virtual(Xd, P, sign=True).double().cpu().numpy()
    refS, _ = chain.sign(X, tables.F_HALF_REFINED, tables.half_kappas(7), lam=lam)
    assert np.linalg.norm(S - refS) / np.linalg.norm(refS) <= {"fp16": 5e-3, "tf32": 5e-3, "bf16": 3e-2}[prec]


@pytest.mark.gpu
def test_rowpanel_virtual_matches_single_gpu_path():
    """Same n, same filter: the row-panel result equals the single-GPU result to rounding (both
    are the same products on the same rounded operands, tiles in another order/assignment)."""
    torch = pytest.importorskip("torch")
    import paper_2507_09165_b200 as pkg
    n = 1536
    X = synth.sdp_shaped(n, 5)
    f = pkg.Filter(pkg.filters.half_filter())
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    a = f.project_rowpanel_virtual(Xd, 4).double().cpu().numpy()
    b = f.project(Xd[None]).double().cpu().numpy()[0]
    assert np.linalg.norm(a - b) / np.linalg.norm(b) < 2e-3


@pytest.mark.gpu
def test_rowpanel_nccl_world1():
    """The real NCCL code path (library communicator, in-place all-gathers of X rows and packed
    tiles) with a world-size-1 process group on this GPU, vs the oracle."""
    torch = pytest.importorskip("torch")
    import torch.distributed as tdist
    import paper_2507_09165_b200 as pkg
    from paper_2507_09165_b200 import dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    tdist.init_process_group("gloo", rank=0, world_size=1)
    try:
        n = 1024
        X = synth.goe(n, 77)
        f = pkg.Filter(pkg.filters.half_filter())
        rp = dist.RowPanelProjector(f, n)
        r0, rows = rp.row_range()
        Xd = torch.tensor(X[r0:r0 + rows], dtype=torch.float32, device="cuda").contiguous()
        out = rp.project(Xd).double().cpu().numpy()
        torch.cuda.synchronize()
        rp.close()
        lam = chain.frobenius_bound(X)
        ref, _ = chain.project(X, tables.F_HALF_REFINED, tables.half_kappas(7), lam=lam)
        assert np.linalg.norm(out - ref[r0:r0 + rows]) / np.linalg.norm(ref) < 5e-3
    finally:
        tdist.destroy_process_group()


# ---------------------------------------------------------------- peer-memory row panels

def _handles_worker(rank, world, port, q):
    import torch.distributed as tdist
    from paper_2507_09165_b200 import dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bytes([rank]) * 64
        got = dist.exchange_ipc_handles(mine)
        q.put((rank, got == [bytes([r]) * 64 for r in range(world)]))
    finally:
        tdist.destroy_process_group()


def test_ipc_handle_exchange_gloo_world2():
    """Setup of the peer-memory path: every rank receives all ranks' 64-byte IPC handles in rank
    order (the bytes psd_rowpanel_p2p_attach consumes), over a gloo world-2 process group."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_handles_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res)


@pytest.mark.gpu
@pytest.mark.parametrize("n,P,prec", [(512, 2, "fp16"), (768, 3, "fp16"), (1024, 4, "tf32"), (2048, 8, "fp16"),
                                      (1024, 1, "bf16")])
def test_rowpanel_p2p_virtual_parity(n, P, prec):
    """Peer-memory row panels (each product kernel stores its tiles into every rank's region,
    epoch barrier between products) with P virtual ranks on one GPU: vs the oracle, exactly
    symmetric, and bit-identical to the NCCL row-panel path (same tiles, same kernel)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2507_09165_b200 as pkg
    X = synth.goe(n, synth.SEED_BASE + n + P)
    f = pkg.Filter(pkg.filters.half_filter(), precision=prec)
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    P_gpu = f.project_rowpanel_p2p_virtual(Xd, P).double().cpu().numpy()
    assert f.status() == "PSD_OK"
    lam = chain.frobenius_bound(X)
    ref, _ = chain.project(X, tables.F_HALF_REFINED, tables.half_kappas(7), lam=lam)
    tol = {"fp16": 5e-3, "tf32": 5e-3, "bf16": 3e-2}[prec]
    assert np.linalg.norm(P_gpu - ref) / np.linalg.norm(ref) <= tol
    assert np.array_equal(P_gpu, P_gpu.T)
    P_nccl = f.project_rowpanel_virtual(Xd, P).double().cpu().numpy()
    assert np.array_equal(P_gpu, P_nccl)
    S = f.project_rowpanel_p2p_virtual(Xd, P, sign=True).double().cpu().numpy()
    refS, _ = chain.sign(X, tables.F_HALF_REFINED, tables.half_kappas(7), lam=lam)
    assert np.linalg.norm(S - refS) / np.linalg.norm(refS) <= tol
    # repeated calls: the epoch counters keep growing, results stay identical
    again = f.project_rowpanel_p2p_virtual(Xd, P).double().cpu().numpy()
    assert np.array_equal(again, P_gpu)


@pytest.mark.gpu
def test_rowpanel_p2p_world1():
    """The real peer-memory code path (region + IPC handle, attach, system-scope epoch barrier
    kernels, owner-row fp32 stores) with a world-size-1 process group on this GPU, vs the oracle."""
    torch = pytest.importorskip("torch")
    import torch.distributed as tdist
    import paper_2507_09165_b200 as pkg
    from paper_2507_09165_b200 import dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    tdist.init_process_group("gloo", rank=0, world_size=1)
    try:
        n = 1024
        X = synth.goe(n, 78)
        f = pkg.Filter(pkg.filters.half_filter())
        rp = dist.PeerRowPanelProjector(f, n)
        r0, rows = rp.row_range()
        Xd = torch.tensor(X[r0:r0 + rows], dtype=torch.float32, device="cuda").contiguous()
        out = rp.project(Xd).double().cpu().numpy()
        out2 = rp.project(Xd).double().cpu().numpy()
        torch.cuda.synchronize()
        rp.close()
        lam = chain.frobenius_bound(X)
        ref, _ = chain.project(X, tables.F_HALF_REFINED, tables.half_kappas(7), lam=lam)
        assert np.linalg.norm(out - ref[r0:r0 + rows]) / np.linalg.norm(ref) < 5e-3
        assert np.array_equal(out, out2)
    finally:
        tdist.destroy_process_group()


def test_bench_spawns_ranks_cpu():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself under
    torch.distributed.run with 2 local ranks (127.0.0.1 rendezvous); rank 0 alone prints the one JSON
    line (here the reference arm, which needs no GPU) with n_gpus = 2 and the same config dict the
    GPU arm prints."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "c3", "--steps", "1", "--warmup", "0", "--ref-seconds", "2"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["filter"] == "c3" and d["config"]["n"] == 1024
    assert d["cpu_baseline"]["cpu_model"] and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
@pytest.mark.parametrize("n,batch,world,prec", [
    (1024, 16, 2, "fp16"),     # CTA-pair kernel for the whole batch and for every shard
    (1024, 24, 3, "fp16x3"),   # split path, K-chunked accumulation
    (512, 6, 4, "fp16"),       # 1-CTA kernel, ragged shards (2, 2, 1, 1)
    (64, 9, 2, "fp16"),        # batched small-n kernel, odd shards
])
def test_batch_shards_bitwise_equal_to_single_gpu(n, batch, world, prec):
    """the c4 partition (contiguous shards of the batch, one per rank, no collective)
    gives every matrix bitwise the result of the single-GPU run of the whole batch."""
    import torch
    from paper_2507_09165_b200 import Filter, filters, dist as pdist
    X = torch.tensor(synth.batch("goe", n, batch, 77 + n), dtype=torch.float32, device="cuda")
    stages = filters.single_filter() if prec.endswith("x3") else filters.half_filter()
    f = Filter(stages, precision=prec)
    full = f.project(X).cpu()
    for rank in range(world):
        first, count = pdist.shard_range(batch, world, rank)
        part = Filter(stages, precision=prec).project(X[first:first + count].contiguous()).cpu()
        assert torch.equal(part, full[first:first + count]), (rank, first, count)

"""world_size-2 gloo tests (CPU) of the multi-GPU host logic: segment sharding, the exact
all-reduce merge of packed occupancy grids, screen tiles and frame assignment."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_09081_b200 import distributed as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, scene_name, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from helpers import Scene
        from oracle import oracle as orc
        orc.set_threads(2)
        sc = Scene(scene_name)
        cn = orc.compute_clip_normals(sc.ls)
        b = D.shard_bounds(sc.ls.n_segments, world)
        part = orc.voxelize(sc.ls, cn, sc.g, r_min=sc.r_min, r_world=sc.r_world,
                            seg_range=(int(b[rank]), int(b[rank + 1])))
        local = torch.from_numpy(part.base.view(np.int32).reshape(-1).copy())
        merged, visited = D.merge_partial_grids(local)
        full = orc.voxelize(sc.ls, cn, sc.g, r_min=sc.r_min, r_world=sc.r_world)
        ok = np.array_equal(merged.numpy().view(np.uint32), full.base.reshape(-1)) and visited == full.visited
        # the partial grids really differ from the merged one (the test would be vacuous otherwise)
        differs = not np.array_equal(part.base, full.base)
        np.save(os.path.join(out_dir, f"ok{rank}.npy"), np.array([ok, differs]))
    finally:
        dist.destroy_process_group()


class OracleEngine:
    """Stand-in for FrameEngine on a host without a GPU: the same `run(cam, grid, r_world, tile, seg_range,
    after_voxelize)` contract and buffers (`wide`, `stats`, `srgb`, `hit_id`), every stage computed by the CPU
    oracle.  It lets the gloo test drive TiledFrame.run / gather_image through a real 2-process exchange."""
    use_wide = True

    def __init__(self, orc, sc):
        self.orc, self.sc = orc, sc
        self.w, self.h = sc.cam.width, sc.cam.height
        self._segs = torch.arange(sc.ls.n_segments, dtype=torch.int32)
        self.stats = torch.zeros(16, dtype=torch.int64)
        self.srgb = torch.zeros((self.h, self.w, 3), dtype=torch.uint8)
        self.hit_id = torch.full((self.h, self.w), -9, dtype=torch.int32)
        self.wide = None
        self.merged_base = None

    def run(self, cam, grid, r_world, tile=None, seg_range=None, after_voxelize=None):
        from types import SimpleNamespace
        orc, sc = self.orc, self.sc
        cn = orc.compute_clip_normals(sc.ls)
        part = orc.voxelize(sc.ls, cn, grid, r_min=sc.r_min, r_world=r_world, seg_range=seg_range)
        self.stats[0] = int(part.visited)
        self.wide = D.widen_packed(torch.from_numpy(part.base.view(np.int32).reshape(-1).copy()))
        if after_voxelize is not None:
            after_voxelize(self)
        packed, _ = D.pack_wide(self.wide)
        self.merged_base = packed.numpy().view(np.uint32).reshape(part.base.shape)
        # the rest of the frame is replicated; this rank keeps only the rows of its tile
        ref = orc.run_frame(sc.ls, grid, r_world, cam, sc.light, strategy=sc.strategy, mode=sc.mode,
                            alpha=sc.alpha, k=sc.k)
        assert np.array_equal(self.merged_base, ref.pyramid.base), "merged grid differs from the whole-set grid"
        x0, y0, x1, y1 = tile
        self.srgb[y0:y1, x0:x1] = torch.from_numpy(ref.image.srgb[y0:y1, x0:x1])
        self.hit_id[y0:y1, x0:x1] = torch.from_numpy(ref.image.hit_id[y0:y1, x0:x1])
        return SimpleNamespace(stats={"voxels_visited": int(self.stats[0])}, stage_ms={"voxelize": 0.0})


def _tiled_worker(rank, world, port, scene_name, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from helpers import Scene
        from oracle import oracle as orc
        orc.set_threads(2)
        sc = Scene(scene_name)
        eng = OracleEngine(orc, sc)
        tf = D.TiledFrame(eng)                       # TorchComm over the gloo group
        assert (tf.rank, tf.world) == (rank, world) and isinstance(tf.comm, D.TorchComm)
        lo, hi = tf.seg_range()
        out = tf.run(sc.cam, sc.g, sc.r_world)
        srgb, hit = tf.gather_image()
        ref = orc.run_frame(sc.ls, sc.g, sc.r_world, sc.cam, sc.light, strategy=sc.strategy, mode=sc.mode,
                            alpha=sc.alpha, k=sc.k)
        ok = out.stats["voxels_visited"] == ref.pyramid.visited
        # thin lines: the 16-byte pre-check lets the ranks exchange the packed words (4 bytes per voxel)
        ok = ok and tf.exchange_kind == "packed" and tf.exchange_bytes == 4 * sc.g.resolution ** 3
        ok = ok and 0 <= lo < hi <= sc.ls.n_segments
        if rank == 0:
            ok = ok and np.array_equal(srgb.numpy(), ref.image.srgb) and np.array_equal(hit.numpy(), ref.image.hit_id)
        else:
            ok = ok and srgb is None and hit is None
        np.save(os.path.join(out_dir, f"tiled{rank}.npy"), np.array([ok, lo, hi]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scene", ["helix32_vsv", "walk32_transp_k2"])
def test_tiled_frame_runs_and_gathers_over_gloo(scene, tmp_path, oracle):
    """TiledFrame.run + gather_image across two real processes (gloo): segment shards, the exact all-reduce
    of the 64-bit accumulators and of the incidence count, per-rank tiles, gather on rank 0."""
    world = 2
    mp.spawn(_tiled_worker, args=(world, _free_port(), scene, str(tmp_path)), nprocs=world, join=True)
    r = [np.load(tmp_path / f"tiled{k}.npy") for k in range(world)]
    assert all(x[0] for x in r)
    assert r[0][1] == 0 and r[0][2] == r[1][1] and r[1][2] > r[1][1]      # the shards tile [0, n)


class PeerComm(D.Comm):
    """A 2-rank job seen from rank 0: all_reduce_sum adds what a peer holding `peer_wide` would contribute to
    whichever of the three buffers of exchange_accumulators is being reduced."""
    rank, world = 0, 2

    def __init__(self, peer_wide):
        self.peer, self.reduced = peer_wide, []

    def all_reduce_sum(self, t):
        if t.numel() == 2 and t.dtype == torch.int64:
            t += D.field_bounds(self.peer).to(t.device); self.reduced.append("bounds")
        elif t.dtype == torch.int32:
            t += D.pack_wide(self.peer.cpu())[0].to(t.device); self.reduced.append("packed")
        else:
            t += self.peer; self.reduced.append("wide")


def test_exchange_accumulators_packed_when_no_field_can_overflow():
    """The multi-GPU exchange: packed 4-byte words while the summed per-rank maxima stay below 2^16,
    else the 8-byte accumulators -- the merged accumulators are the plain sum either way."""
    g = torch.Generator().manual_seed(3)
    cnt_a = torch.randint(0, 300, (4096,), generator=g); occ_a = torch.randint(0, 30000, (4096,), generator=g)
    cnt_b = torch.randint(0, 300, (4096,), generator=g); occ_b = torch.randint(0, 30000, (4096,), generator=g)
    a = (cnt_a << 32) | occ_a
    b = (cnt_b << 32) | occ_b
    mine = a.clone()
    comm = PeerComm(b)
    nbytes, kind = D.exchange_accumulators(mine, comm)
    assert (nbytes, kind) == (4 * 4096, "packed") and comm.reduced == ["bounds", "packed"]
    assert torch.equal(mine, a + b)
    # one voxel whose occupancy sums COULD reach 2^16 (40000 here, 30000 somewhere on the peer): the bound fails
    a2 = a.clone(); a2[7] = (5 << 32) | 40000
    mine = a2.clone()
    comm = PeerComm(b)
    nbytes, kind = D.exchange_accumulators(mine, comm)
    assert (nbytes, kind) == (8 * 4096, "wide") and comm.reduced == ["bounds", "wide"]
    assert torch.equal(mine, a2 + b)
    # counts near the field limit: 40000 + 299 < 65536 is fine, and the packed words then have their top bit set
    a3 = a.clone(); a3[11] = (40000 << 32) | 17
    mine = a3.clone()
    nbytes, kind = D.exchange_accumulators(mine, PeerComm(b))
    assert kind == "packed" and torch.equal(mine, a3 + b)


def test_emulated_comm_contract():
    c = D.EmulatedComm(1, 4)
    assert (c.rank, c.world) == (1, 4) and c.gather(torch.zeros(1)) is None
    with pytest.raises(RuntimeError):
        c.all_reduce_sum(torch.zeros(1))
    with pytest.raises(ValueError):
        D.EmulatedComm(4, 4)
    seen = []
    c.peers = seen.append
    t = torch.ones(2)
    c.all_reduce_sum(t)
    assert seen and seen[0] is t
    one = D.Comm()
    assert (one.rank, one.world) == (0, 1) and one.gather(t) == [t]


@pytest.mark.parametrize("scene", ["helix64_vcsv", "diag_vcsv"])   # diag: 16-bit occupancy saturates
def test_sharded_voxelize_merge_gloo(scene, tmp_path, oracle):
    world = 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, scene, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        ok, differs = np.load(tmp_path / f"ok{r}.npy")
        assert ok and differs


def test_widen_pack_roundtrip_and_saturation():
    base = np.array([0, (3 << 16) | 100, (0xFFFF << 16) | 0xFFFF, (40000 << 16) | 50000], dtype=np.uint32)
    t = torch.from_numpy(base.view(np.int32).copy())
    wide = D.widen_packed(t)
    assert wide.tolist() == [0, (3 << 32) | 100, (0xFFFF << 32) | 0xFFFF, (40000 << 32) | 50000]
    packed, visited = D.pack_wide(wide)
    assert np.array_equal(packed.numpy().view(np.uint32), base) and visited == 3 + 0xFFFF + 40000
    # two ranks holding the last word: both fields must saturate separately, no carry between them
    packed2, visited2 = D.pack_wide(wide + wide)
    want = np.array([0, (6 << 16) | 200, (0xFFFF << 16) | 0xFFFF, (0xFFFF << 16) | 0xFFFF], dtype=np.uint32)
    assert np.array_equal(packed2.numpy().view(np.uint32), want) and visited2 == 2 * visited


@pytest.mark.parametrize("n,world", [(0, 4), (1, 4), (10, 3), (1000003, 8), (7, 8)])
def test_shard_bounds_cover(n, world):
    b = D.shard_bounds(n, world)
    assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
    assert len(b) - 1 == max(1, min(world, max(1, n)))


@pytest.mark.parametrize("w,h,world", [(1920, 1080, 1), (1920, 1080, 8), (64, 37, 4), (5, 3, 8)])
def test_tiles_partition_the_image(w, h, world):
    seen = np.zeros((h, w), dtype=np.int32)
    for x0, y0, x1, y1 in D.tile_rects(w, h, world):
        assert 0 <= x0 <= x1 <= w and 0 <= y0 <= y1 <= h
        seen[y0:y1, x0:x1] += 1
    assert (seen == 1).all()


def test_frames_for_rank_partition():
    frames = sorted(f for r in range(8) for f in D.frames_for_rank(100, r, 8))
    assert frames == list(range(100))


def test_balanced_rows():
    rows = [0, 135, 270, 405, 540, 675, 810, 945, 1080]
    w = [2.0, 3.8, 4.2, 4.4, 4.9, 4.7, 3.2, 1.9]
    b = D.balanced_rows(rows, w, 1080)
    assert b[0] == 0 and b[-1] == 1080 and all(b[i + 1] > b[i] for i in range(8))
    # the work each new strip would have held under the piecewise-constant density is equal to within a row's worth
    dens = np.repeat(np.array(w) / 135.0, 135)
    share = [dens[b[i]:b[i + 1]].sum() for i in range(8)]
    assert max(share) - min(share) <= 2 * dens.max()
    assert b[1] - b[0] > 135 and b[4] - b[3] < 135          # light strips grow, heavy strips shrink
    assert D.balanced_rows([0, 540, 1080], [1, 1], 1080) == [0, 540, 1080]
    assert D.balanced_rows([0, 540, 1080], [0, 0], 1080) == [0, 540, 1080]    # nothing measured: equal strips
    assert D.balanced_rows([0, 1, 3], [5, 0], 3) == [0, 1, 3]                    # every strip keeps a row
    assert D.balanced_rows([0, 2, 3], [0, 9], 3) == [0, 2, 3]


def test_tiled_frame_set_rows_validation():
    class E:
        w, h = 64, 48
        _segs = torch.arange(10, dtype=torch.int32)
    tf = D.TiledFrame(E(), comm=D.EmulatedComm(1, 3))
    assert tf.rows() == [0, 16, 32, 48]
    tf.set_rows([0, 5, 40, 48])
    assert tf.tiles[1] == (0, 5, 64, 40) and tf.rows() == [0, 5, 40, 48]
    for bad in ([0, 5, 48], [0, 5, 5, 48], [1, 5, 40, 48], [0, 5, 40, 47]):
        with pytest.raises(ValueError):
            tf.set_rows(bad)
    assert tf.rebalance(3.0) == [0, 5, 40, 48]        # an emulated rank alone cannot rebalance
    one = D.TiledFrame(E(), comm=D.Comm())
    assert one.rebalance(1.0) == [0, 48]

"""the reference's own front ends -- `linevox render` (lv/cli.py:66-80) and the websocket
frame server (lv/server.py:43-117) -- driving the B200 pipeline UNCHANGED.  The unmodified reference package
(pip-installed into baseline/_ref by __graft_entry__.build()) is imported, its `ScenePipeline` name is pointed
at `paper_2510_09081_b200.ScenePipeline`, and its CLI / server code runs as it is: the files it writes and the
frames it streams must be byte-identical to what the same front end produces with the reference's own CPU
pipeline.  Skipped where baseline/_ref or numba is absent."""
import asyncio
import hashlib
import json
import os
import socket
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "linevox")):
        pytest.skip("baseline/_ref (the pip-installed reference package) is not present")
    try:
        import numba  # noqa: F401
        import websockets  # noqa: F401
    except Exception as e:
        pytest.skip(f"the reference package's dependencies are missing: {e}")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "lvx_numba_cache"))
    sys.path.insert(0, REF)
    import linevox
    import linevox.cli
    import linevox.pipeline
    import linevox.server
    return linevox


@pytest.fixture(scope="module")
def lvx():
    from paper_2510_09081_b200 import _native
    _native.require_cuda()
    import paper_2510_09081_b200 as m
    return m


def sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("argv", [
    ["--input", "gen:random_streamlines?polylines=40&verts_per_line=60", "--res", "64", "--strategy", "vcsv",
     "--width", "160", "--height", "120", "--dump"],
    ["--input", "gen:helix?turns=3&verts=90", "--res", "32", "--strategy", "vsv", "--mode", "transparent",
     "--alpha", "0.4", "--k", "4", "--width", "96", "--height", "96", "--r", "0.5", "--dump"],
])
def test_reference_cli_render_runs_on_the_gpu_pipeline(ref, lvx, argv, tmp_path, monkeypatch):
    cpu, gpu = str(tmp_path / "cpu"), str(tmp_path / "gpu")
    assert ref.cli.main(["render", *argv, "--out", cpu]) == 0                 # the reference as it is (numba, CPU)
    monkeypatch.setattr(ref.pipeline, "ScenePipeline", lvx.ScenePipeline)      # cmd_render imports the name at call time
    assert ref.cli.main(["render", *argv, "--out", gpu]) == 0                 # same front end, B200 pipeline
    for ext in (".ppm", ".hiti", ".voxp", ".abuf") + ((".culp",) if "vcsv" in argv else ()):
        assert os.path.getsize(gpu + ext) > 0
        assert sha(gpu + ext) == sha(cpu + ext), f"{ext} written through the reference CLI differs"
    keys = lambda p: sorted(line.split("=")[0] for line in open(p + ".stats.txt").read().split())
    assert keys(gpu) == keys(cpu)
    stat = lambda p: dict(line.split("=") for line in open(p + ".stats.txt").read().split())
    for k in ("segments", "vertices", "resolution", "voxels_visited", "fragments", "fragment_touches", "ray_capsule_tests"):
        assert stat(gpu)[k] == stat(cpu)[k], k


def test_reference_server_streams_gpu_frames(ref, lvx, monkeypatch):
    """lv/server.py:43-117 with its ScenePipeline pointed at the GPU one: pose messages in, frame_header + sRGB
    body out; a `set` of a view setting and of a geometry setting (which makes the server call build_geometry)
    in between.  Every streamed frame equals the reference pipeline's frame for the same pose and settings."""
    import websockets
    port = _free_port()
    kw = dict(input="gen:random_streamlines?polylines=30&verts_per_line=40", res=32, strategy="vcsv", width=96,
              height=64, port=port)
    poses = [dict(position=[60.0, 40.0, 45.0], forward=[-1.0, -0.6, -0.5], up=[0.0, 0.0, 1.0]),
             dict(position=[10.0, 70.0, 30.0], forward=[0.3, -1.0, -0.2], up=[0.0, 0.0, 1.0], fov=0.9)]

    def reference_frames():
        out = []
        cfg = ref.PipelineConfig(**kw)
        pipe = ref.ScenePipeline(cfg)
        cam = lambda p: ref.Camera(np.array(p["position"]), np.array(p["forward"]), np.array(p["up"]),
                                   fov=float(p.get("fov", np.deg2rad(cfg.cam_fov))), width=cfg.width, height=cfg.height)
        out.append(pipe.render_frame(cam(poses[0])).srgb_bytes())
        pipe.cfg = ref.PipelineConfig.from_sources(None, {**kw, "light": "0.2,-0.9,-0.4"})
        out.append(pipe.render_frame(cam(poses[1])).srgb_bytes())
        pipe.cfg = ref.PipelineConfig.from_sources(None, {**kw, "light": "0.2,-0.9,-0.4", "r": 0.45})
        pipe.build_geometry()
        out.append(pipe.render_frame(cam(poses[1])).srgb_bytes())
        return out, dict(pipe.stats)

    want, ref_stats = reference_frames()
    monkeypatch.setattr(ref.server, "ScenePipeline", lvx.ScenePipeline)

    async def session():
        ready = asyncio.Event()
        task = asyncio.create_task(ref.server.serve_forever(ref.PipelineConfig(**kw), ready))
        await asyncio.wait_for(ready.wait(), 60)
        got = []
        try:
            async with websockets.connect(f"ws://127.0.0.1:{port}", max_size=None) as ws:
                async def frame(pose, pid):
                    await ws.send(json.dumps({"type": "pose", "id": pid, **pose}))
                    hdr = json.loads(await asyncio.wait_for(ws.recv(), 120))
                    assert hdr["type"] == "frame_header", hdr
                    body = await asyncio.wait_for(ws.recv(), 120)
                    return hdr, body
                got.append(await frame(poses[0], 11))
                await ws.send(json.dumps({"type": "set", "key": "light", "value": "0.2,-0.9,-0.4"}))
                got.append(await frame(poses[1], 12))
                await ws.send(json.dumps({"type": "set", "key": "r", "value": 0.45}))      # geometry key: rebuild
                got.append(await frame(poses[1], 13))
                await ws.send(json.dumps({"type": "set", "key": "res", "value": 33}))       # invalid: error, not a crash
                err = json.loads(await asyncio.wait_for(ws.recv(), 60))
                assert err["type"] == "error"
        finally:
            task.cancel()
            try:
                await task
            except (asyncio.CancelledError, Exception):
                pass
        return got

    got = asyncio.run(session())
    for i, ((hdr, body), w) in enumerate(zip(got, want)):
        assert (hdr["width"], hdr["height"], hdr["id"]) == (96, 64, i + 1) and hdr["pose_id"] == 11 + i
        assert isinstance(body, bytes) and len(body) == 96 * 64 * 3
        assert body == w, f"streamed frame {i} differs from the reference pipeline's frame"
    last = got[-1][0]["stats"]
    assert sorted(last) == sorted(ref_stats)
    for k in ("segments", "vertices", "resolution", "voxels_visited", "fragments", "ray_capsule_tests"):
        assert last[k] == ref_stats[k], k

"""Service frame path (service.py mirror): request
validation, payload framing, HTTP routes and the latest-wins stream (CPU,
injected renderer); GPU: the u8 kernel epilogue equals Frame.rgb8 and the
PNG round-trips."""

import asyncio
import io
import json
import os
import threading
import time

import numpy as np
import pytest

from conftest import golden_grid

REF_SRC = "/root/reference/pkg/src"

BODIES = [
    {"eye": [1, 1, 1], "look": [2, 1, 1]},
    {"eye": [1, 1, 1], "look": [2, 1, 1], "fov": 75, "width": 64, "height": 32},
    {"eye": [1, 1, 1], "look": [1, 1, 1]},
    {"eye": [1, 1], "look": [2, 1, 1]},
    {"eye": [1, 1, float("nan")], "look": [2, 1, 1]},
    {"eye": [1, 1, 1], "look": [2, 1, "x"]},
    {"eye": [1, 1, 1], "look": [2, 1, 1], "fov": 180},
    {"eye": [1, 1, 1], "look": [2, 1, 1], "width": 0},
    {"eye": [1, 1, 1], "look": [2, 1, 1], "height": 5000},
    {"eye": [1, 1, 1], "look": [2, 1, 1], "width": 3.0},
    {"eye": [True, 1, 1], "look": [2, 1, 1]},
    [1, 2, 3],
]


def _parse(mod, body, **kw):
    try:
        c = mod.parse_camera(body, **kw)
        return ("ok", tuple(c.eye), tuple(np.asarray(c.forward, float)),
                c.vfov_deg, c.width, c.height)
    except ValueError as exc:
        return ("err", str(exc))


def test_parse_camera_messages():
    from paper_2507_14624_b200 import service
    got = [_parse(service, b) for b in BODIES]
    assert got[0][0] == "ok" and got[0][4:] == (512, 512)
    assert got[1][3:] == (75.0, 64, 32)
    assert got[2] == ("err", "look: must differ from eye")
    assert got[3] == ("err", "eye: expected 3 finite numbers")
    assert got[6] == ("err", "fov: expected a number in (0, 180)")
    assert got[7] == ("err", "width: expected an integer in [1, 4096]")
    assert got[11] == ("err", "camera: request body must be a JSON object")


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present")
def test_parse_camera_matches_reference():
    import subprocess
    import sys
    code = ("import json,sys,numpy as np\n"
            "sys.path.insert(0, %r)\n"
            "from lfprobe import service\n"
            "bodies = json.loads(sys.stdin.read())\n"
            "out = []\n"
            "for b in bodies:\n"
            "    try:\n"
            "        c = service.parse_camera(b)\n"
            "        out.append(['ok', list(c.eye), [float(x) for x in c.forward],"
            " c.vfov_deg, c.width, c.height])\n"
            "    except ValueError as e:\n"
            "        out.append(['err', str(e)])\n"
            "print(json.dumps(out))\n" % REF_SRC)
    body = json.dumps(BODIES).replace("NaN", "NaN")
    env = dict(os.environ, NUMBA_CACHE_DIR="/tmp/numba_cache")
    r = subprocess.run([sys.executable, "-c", code], input=body, text=True,
                       capture_output=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr
    ref = json.loads(r.stdout)
    from paper_2507_14624_b200 import service
    for b, want in zip(BODIES, ref):
        got = _parse(service, b)
        if want[0] == "err":
            assert got == tuple(want), b
        else:
            assert got[0] == "ok" and list(got[1]) == want[1], b
            assert list(got[2]) == want[2] and got[3:] == tuple(want[3:]), b


def test_frame_payload_and_png():
    from PIL import Image

    from paper_2507_14624_b200 import service
    assert service.frame_payload(258, b"xy") == b"\x00\x00\x01\x02xy"
    img = (np.arange(4 * 5 * 3) % 256).astype(np.uint8).reshape(4, 5, 3)
    png = service.encode_png(img)
    back = np.asarray(Image.open(io.BytesIO(png)).convert("RGB"))
    assert np.array_equal(back, img)


class _Grid:
    dims = (2, 2, 2)
    bounds = (np.zeros(3), np.ones(3))


def _fake_render(delay=0.0, log=None):
    from paper_2507_14624_b200 import service

    def render(grid, cam):
        if delay:
            time.sleep(delay)
        if log is not None:
            log.append(cam)
        img = np.full((cam.height, cam.width, 3), 7, np.uint8)
        return service.encode_png(img), {"traceMs": 0.5, "missFraction": 0.25,
                                         "unknownFraction": 0.0}
    return render


def test_http_routes():
    from fastapi.testclient import TestClient

    from paper_2507_14624_b200 import service
    app = service.create_app(scenes={"room": {"id": "room", "name": "Room",
                                              "grid": _Grid()}},
                             render=_fake_render())
    c = TestClient(app)
    d = c.get("/scenes").json()
    assert d == [{"id": "room", "name": "Room", "probeCount": 8,
                  "gridDims": [2, 2, 2],
                  "bounds": {"lo": [0.0, 0.0, 0.0], "hi": [1.0, 1.0, 1.0]}}]
    r = c.post("/scenes/room/render", json={"eye": [0, 0, 0], "look": [1, 0, 0],
                                           "width": 8, "height": 4})
    assert r.status_code == 200 and r.headers["content-type"] == "image/png"
    assert json.loads(r.headers["X-Render-Stats"])["missFraction"] == 0.25
    assert c.post("/scenes/room/render", json={"eye": [0, 0, 0]}).status_code == 400
    assert c.post("/scenes/nope/render", json={}).status_code == 404


def test_websocket_stream_and_errors():
    from fastapi.testclient import TestClient

    from paper_2507_14624_b200 import service
    app = service.create_app(scenes={"room": {"id": "room", "name": "Room",
                                              "grid": _Grid()}},
                             render=_fake_render())
    c = TestClient(app)
    with c.websocket_connect("/scenes/nope/stream") as ws:
        assert "unknown scene" in json.loads(ws.receive_text())["error"]
    with c.websocket_connect("/scenes/room/stream") as ws:
        ws.send_text("not json")
        assert "error" in json.loads(ws.receive_text())
        spec = {"eye": [0, 0, 0], "look": [0, 0, 1], "width": 6, "height": 6}
        ws.send_text(json.dumps(spec))
        head = json.loads(ws.receive_text())
        assert head["frameCounter"] == 1 and head["camera"] == spec
        payload = ws.receive_bytes()
        assert payload[:4] == (1).to_bytes(4, "big")
        assert payload[4:12] == b"\x89PNG\r\n\x1a\n"


def test_latest_wins_collapses_pending_cameras():
    from paper_2507_14624_b200 import service
    sent = []
    gate = threading.Event()

    def render(cam):
        gate.wait(5)
        return b"png", {"traceMs": 0.0}

    async def send(counter, spec, png, stats):
        sent.append((counter, spec))

    async def main():
        s = service.LatestWinsSession(render, send)
        task = asyncio.create_task(s.run())
        s.submit("cam0", 0)
        await asyncio.sleep(0.05)          # frame 0 is rendering (gated)
        for k in range(1, 6):
            s.submit(f"cam{k}", k)         # collapse into the newest
        gate.set()
        while len(sent) < 2:
            await asyncio.sleep(0.01)
        s.close()
        await asyncio.wait_for(task, 5)
        return s

    s = asyncio.run(main())
    assert sent == [(1, 0), (2, 5)]
    assert s.dropped == 4


@pytest.mark.gpu
def test_gpu_rgb8_epilogue_and_png(golden):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    import __graft_entry__
    __graft_entry__.build()
    from PIL import Image

    from paper_2507_14624_b200 import render, service
    from paper_2507_14624_b200.grid import ProbeHierarchy
    z = golden("pcgrid")
    g = golden_grid(z)
    cams = [render.Camera(eye=(1.3, 1.1, 1.7), forward=(0.4, -0.2, -1.0),
                          width=96, height=80),
            render.Camera(eye=(0.5, 0.25, 0.5), forward=(1.0, 0.5, 0.7),
                          width=33, height=17)]
    for src in (g, ProbeHierarchy([g])):
        for cam in cams:
            fr = render.render_frame(src, cam)
            rgb8, st, stats = render.render_frame_rgb8(src, cam)
            assert np.array_equal(rgb8, fr.rgb8)
            assert np.array_equal(st, fr.status)
            png, pub = service.render_png(src, cam)
            back = np.asarray(Image.open(io.BytesIO(png)).convert("RGB"))
            assert np.array_equal(back, fr.rgb8)
            assert pub["missFraction"] == fr.stats["missFraction"]
    # non-grid sources (single probe / probe list) through the same epilogue
    from paper_2507_14624_b200.grid import MapChain, ProbeData
    ps = g.probe_set
    probes = [ProbeData(ps.origins[i], MapChain(ps.irr_hi[i], ps.dist_hi[i],
                                                ps.dir_hi[i], ps.dist_lo[i]),
                        np.zeros(3), np.full(3, 3.0)) for i in range(3)]
    for src in (probes[0], probes):
        fr = render.render_frame(src, cams[0])
        rgb8, _, _ = render.render_frame_rgb8(src, cams[0])
        assert np.array_equal(rgb8, fr.rgb8)

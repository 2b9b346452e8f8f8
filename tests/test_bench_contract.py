"""bench.py's contract on CPU: workloads, the oracle-only reference arm, layouts.

* bench.WORKLOADS (restated so the reference arm needs no product import)
  equals paper_2504_06095_b200.workloads.SHAPES;
* the oracle's pair layout (its own shard map) equals the product's arena
  layout -- bench --check and the full-size parity tests slice the device
  arenas with it;
* ``bench.py --impl reference`` runs the full workload per step on the oracle
  and never imports or loads the product library, and prints the same config
  object as our arm.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import bench
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_workloads_match_product_shapes():
    from paper_2504_06095_b200.workloads import SHAPES
    assert set(SHAPES) == set(bench.WORKLOADS)
    for name, s in SHAPES.items():
        hidden, ffn, heads, layers = bench.WORKLOADS[name][:4]
        assert (s.hidden, s.ffn, s.heads, s.layers) == (hidden, ffn, heads, layers)
        assert s.elems() == bench.workload_elems(name)


@pytest.mark.parametrize("name,layers", [("gpt-1.3b", 2), ("llama3-8b-shaped", 1),
                                         ("mlp-h1024-ffn4096", 1)])
@pytest.mark.parametrize("n1,n2", [(4, 3), (4, 2), (2, 1)])
def test_oracle_layout_equals_product_layout(name, layers, n1, n2):
    from paper_2504_06095_b200.workloads import SHAPES, pair_layout
    hidden, ffn, heads = bench.WORKLOADS[name][:3]
    segs, h_elems, r_elems = O.pair_layout(hidden, ffn, heads, layers, n1, n2)
    lay = pair_layout(SHAPES[name], n1, n2, layers=layers)
    assert h_elems == list(lay.h_elems) and r_elems == list(lay.r_elems)
    assert len(segs) == len(lay.segs)
    for (k, unit, comp, sync, hc, rc, hb, rb), (k2, u2, hc2, rc2, hb2, rb2) in zip(segs, lay.segs):
        assert (k, unit) == (k2, u2)
        assert all(np.array_equal(a, b) for a, b in zip(hc, hc2))
        assert all(np.array_equal(a, b) for a, b in zip(rc, rc2))
        assert np.array_equal(hb, hb2) and np.array_equal(rb, rb2)


def test_check_pair_segment_flags_errors():
    """The checker itself: exact outputs pass, a perturbed unit fails, and a
    unit whose two copies differ is reported as not bit-identical."""
    segs, h_elems, r_elems = O.pair_layout(64, 96, 0, 1, 4, 3)
    seg = segs[0]
    rng = np.random.default_rng(0)
    h = [rng.standard_normal(e) for e in h_elems]
    r = [rng.standard_normal(e) for e in r_elems]
    hv, rv = O.segment_views(seg, h, r)
    ho, ro = [x.copy() for x in hv], [x.copy() for x in rv]
    O.nonuniform_sync(seg[2], seg[3], seg[4], seg[5], ho, ro, seg[1], op=O.OP_WEIGHTED,
                      weights=(bench.W_H, bench.W_R))
    err, same = O.check_pair_segment(seg, hv, rv, ho, ro, (bench.W_H, bench.W_R))
    assert err == 0.0 and same
    ro[0][5] += 1.0
    err, same = O.check_pair_segment(seg, hv, rv, ho, ro, (bench.W_H, bench.W_R))
    assert err > 1e-3 and not same


def test_reference_arm_is_oracle_only_and_same_config():
    code = (
        "import sys, json, io, contextlib\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "import bench\n"
        "buf = io.StringIO()\n"
        "with contextlib.redirect_stdout(buf):\n"
        "    bench.main(['--impl', 'reference', '--workload', 'mlp-h1024-ffn4096',\n"
        "                '--steps', '2', '--warmup', '1'])\n"
        "line = json.loads(buf.getvalue().strip().splitlines()[-1])\n"
        "mods = sorted(m for m in sys.modules if m.startswith('paper_2504_06095_b200'))\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'line': line, 'mods': mods, 'libntp_b200': 'libntp_b200' in maps,\n"
        "                  'oracle': 'libntp_oracle' in maps}))\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["mods"] == [] and not res["libntp_b200"] and res["oracle"], res
    line = res["line"]
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["config"] == bench.workload_config("mlp-h1024-ffn4096", 1)
    assert line["unit"] == "GB/s" and line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    # one step = the whole workload: value = replica gradient bytes / step time
    S = bench.workload_elems("mlp-h1024-ffn4096") * 4
    assert abs(line["value"] - S / (line["ms_per_step"] * 1e-3) / 1e9) < 0.01 * line["value"]


def test_reexec_under_torchrun(monkeypatch):
    """`python bench.py --gpus 4` outside torchrun relaunches under
    torch.distributed.run with 4 processes on a 127.0.0.1 rendezvous."""
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    assert bench.main(["--gpus", "4", "--steps", "3", "--warmup", "3"]) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "3", "--warmup", "3"]
    assert cmd[-7].endswith("bench.py")

"""Host-side pieces of bench.py that run without a GPU.

* The reference arm (`--impl reference`) runs the reference's own CPU path
  and must not load the product: paper_2011_01805_b200 is never imported and
  libtiletensor_b200.so never mapped in that process.
* The e2e host-staging guard picks the largest slab that fits, and reports 0
  (e2e skipped) when not even 1/8 of the input fits.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def test_reference_arm_does_not_load_the_product():
    ref = ROOT / "oracle" / "_ref" / "libttref.so"
    if not ref.exists():
        pytest.skip("oracle/_ref not built")
    code = (
        "import sys, json; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0',"
        "'--ref-slab-tiles','1']; import bench; bench.main();"
        "maps=open('/proc/self/maps').read();"
        "print(json.dumps({'mods': [m for m in sys.modules if m.startswith('paper_2011_01805_b200')],"
        "'product_so': 'libtiletensor_b200' in maps, 'ref_so': 'libttref.so' in maps}))")
    proc = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                          timeout=600)
    assert proc.returncode == 0, proc.stderr[-2000:]
    lines = [json.loads(ln) for ln in proc.stdout.splitlines() if ln.startswith("{")]
    line, probe = lines[0], lines[1]
    assert probe == {"mods": [], "product_so": False, "ref_so": True}
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["config"]["global_x"] == [2048, 2048, 512]
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    one = line["cpu_baseline"]["one_thread"]
    assert one["cores"] == 1 and one["value"] > 0


def test_reference_arm_config_matches_gpu_arm():
    import bench
    for world in (1, 2, 8):
        cfg = bench.workload_config(world, bench.resolve_scaling(type("A", (), {"scaling": "auto"}), world))
        assert cfg["global_x"] == [2048, 2048, 512]
    assert bench.workload_config(4, "weak")["global_x"] == [8192, 2048, 512]


def test_host_slab_fraction(monkeypatch):
    import bench
    n = 2048 * 2048 * 512
    for gib, frac in ((200, 1.0), (20, 0.5), (10, 0.25), (5, 0.125), (2, 0.0)):
        monkeypatch.setenv("TT_BENCH_HOST_GIB", str(gib))
        monkeypatch.setenv("LOCAL_WORLD_SIZE", "1")
        assert bench.host_slab_fraction(n, 1, None, None) == frac, gib

"""bench.py contract pieces that run without a GPU: the reference arm's JSON
line (the C oracle on host cores) and the ray-block sharding."""
import json
import subprocess
import sys

import numpy as np

from conftest import ROOT


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--config", "c1", "--res", "64x64", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] in ("port", "reference")


def test_shard_contiguous_blocks():
    sys.path.insert(0, str(ROOT))
    import bench
    wave = ("primary", "primary", True, np.zeros((10, 3)), np.zeros((10, 3)), np.zeros(10),
            np.ones(10))
    parts = [bench.shard(wave, r, 3) for r in range(3)]
    assert sum(p[3].shape[0] for p in parts) == 10
    assert [p[3].shape[0] for p in parts] == [3, 3, 4]

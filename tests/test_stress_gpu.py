"""FT-heavy co-serving stress with a watchdog (keep the configuration that exposed
the round-1 stall in the default coverage).  The 8B-shaped bench loop at 4 and 10 req/s (the
low rates leave most of every iteration to finetuning windows, many of them multi-window
backward iterations) runs in a subprocess under a timeout: a hang fails the test instead of
the suite, and a kernel whose mbarrier wait exceeds 20 s traps (common.cuh) rather than spin."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ft_heavy_side_rates_complete():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--rate", "10", "--rates", "4,10",
           "--steps", "150", "--warmup", "5", "--no-cpu-baseline", "--kernel-profile", "0"]
    try:
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    except subprocess.TimeoutExpired:
        pytest.fail("co-serving loop did not finish within 900 s (stall)")
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["value"] > 0 and "4" in line["other_rates"]
    assert line["other_rates"]["4"]["value"] > 0
    # every decoding request keeps streaming: inter-token latency stays near the SLO
    assert line["inference"]["itl_samples"] > 0
    assert line["inference"]["itl_p99_ms"] < 1.5 * line["inference"]["slo_ms"]

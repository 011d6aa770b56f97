"""Host-side pieces of bench.py that need no GPU."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_watchdog_turns_a_stuck_multi_rank_run_into_an_error():
    # a rank whose neighbour never arrives must exit non-zero, not block
    code = ("import sys, time; sys.path.insert(0, %r); import bench; "
            "bench.arm_watchdog(1); time.sleep(30)" % str(ROOT))
    env = dict(os.environ, HJB_BENCH_WATCHDOG_S="0.5")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=25)
    assert p.returncode == 3
    assert "watchdog" in json.loads(p.stdout.strip().splitlines()[-1])["error"]


def test_watchdog_cancelled_run_exits_normally():
    sys.path.insert(0, str(ROOT))
    import bench
    t = bench.arm_watchdog(0)
    t.cancel()
    assert not t.is_alive() or t.finished.is_set()

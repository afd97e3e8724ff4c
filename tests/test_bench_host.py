"""Host logic of bench.py that needs no GPU: the clock sampler's timed-region window and the argument
contract of the driver's commands."""
import importlib.util
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_clock_sampler_reports_only_the_timed_region():
    b = _bench()
    c = b.ClockSampler(0)
    row = lambda t, mhz, cap: [t, str(mhz), "1965", "Not Active", "Not Active", "Not Active", cap]
    # warm-up samples (one throttled by a thermal event that must not leak into the report), the timed
    # region [10, 20], and samples after it
    c.samples = [row(1.0, 1200, "Not Active"), [2.0, "1300", "1965", "Active", "Not Active", "Not Active", "Not Active"],
                 row(9.0, 1950, "Not Active"), row(12.0, 1965, "Active"), row(15.0, 1965, "Not Active"),
                 row(25.0, 500, "Not Active")]
    c._t0, c._t1 = 10.0, 20.0
    s = c.summary()
    assert s["n_samples"] == 3                      # the last one before the region + the two inside
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]         # hw_slowdown during warm-up is outside the window
    c.samples = []
    assert c.summary()["reasons"] == ["unsampled"]


def test_reference_arm_other_ranks_exit_without_work():
    """`bench.py --impl reference` under torchrun: ranks other than 0 print nothing and exit 0."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                         env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == ""

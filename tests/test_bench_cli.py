"""bench.py's command line on a CPU-only host: the reference arm (the
reference's own run_contour -- the unmodified package from baseline/_ref when
installed, else the oracle port -- on the host cores) prints one JSON line
with the contract's keys and never loads the product library; --help
parses; --gpus N re-launches under torch.distributed.run."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# run the reference arm in-process, then report which shared objects it mapped
_PROBE = """
import json, sys
sys.argv = ["bench.py", "--impl", "reference", "--config", "er", "--steps", "2", "--warmup", "1"]
sys.path.insert(0, {root!r})
import bench
bench.main()
maps = open("/proc/self/maps").read()
print("MAPS " + json.dumps(sorted({{l.split()[-1] for l in maps.splitlines() if l.endswith(".so")}})))
"""


def test_reference_arm_prints_contract_line_without_product_library():
    out = subprocess.run([sys.executable, "-c", _PROBE.format(root=ROOT)], capture_output=True,
                         text=True, timeout=600, cwd=ROOT, check=True).stdout
    line = json.loads([x for x in out.splitlines() if x.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "edges/s" and line["value"] > 0
    for key in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["steps"] == 2 and line["reference_sweeps"]["executed"] >= 1
    maps = json.loads([x for x in out.splitlines() if x.startswith("MAPS ")][-1][5:])
    assert not [p for p in maps if "libcontour" in p], maps


def test_both_arms_share_the_config_object():
    sys.path.insert(0, ROOT)
    import bench
    n, m = bench.sizes_of("rmat28")
    assert (n, m) == (1 << 28, 8_589_934_592)
    a = bench.shared_config("rmat28", n, m, True)
    assert a == bench.shared_config("rmat28", n, m, True)
    assert a["workload"].startswith("configs[4]")
    assert bench.parse([]).config == "rmat28"  # the north-star config is the default


def test_help_parses():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, check=True).stdout
    assert "--impl" in out and "--gpus" in out and "--exchange" in out


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8", "--steps", "3"])
    args = bench.parse(["--gpus", "8", "--steps", "3"])
    assert bench.relaunch(args) == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "8", "--steps", "3"][1:] or cmd[-4:] == ["--gpus", "8", "--steps", "3"]

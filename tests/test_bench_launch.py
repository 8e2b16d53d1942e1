"""bench.py's own launcher: --gpus N re-launches under torchrun, one rank per GPU,
and fails loudly when fewer GPUs are visible; the reference arm stays product-free."""

import json
import os
import subprocess
import sys

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_torchrun_command_shape():
    cmd = bench.torchrun_command(4, ["--gpus", "4", "--steps", "2"], port=29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[cmd.index("--master-port") + 1] == "29555"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"] and cmd[-5].endswith("bench.py")


def test_relaunch_refuses_without_enough_gpus(capsys):
    called = []
    rc = bench.relaunch_under_torchrun(8, ["--gpus", "8"], count=lambda: 1, run=lambda *a, **k: called.append(a) or 0)
    assert rc == 2 and not called
    assert "only 1 CUDA device" in capsys.readouterr().err


def test_relaunch_spawns_one_rank_per_gpu():
    seen = {}

    def fake_run(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    assert bench.relaunch_under_torchrun(2, ["--gpus", "2"], count=lambda: 8, run=fake_run) == 0
    assert "--nproc-per-node=2" in seen["cmd"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], env=env, capture_output=True,
                       text=True)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr


def test_reference_arm_is_product_free_and_real():
    """cfg0 through the reference arm: a real (time-boxed) CPU step, no product import,
    no repo .so mapped, and ms_per_step equal to the wall time of the work done."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "0",
                        "--ref-box", "60"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["product_imported"] is False and d["repo_so_mapped"] == []
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["iterations"] >= 5
    assert abs(d["value"] - d["config"]["ndof"] * cb["iterations"] / cb["wall_s"]) <= 1e-6 * d["value"]
    assert abs(d["ms_per_step"] - 1e3 * cb["wall_s"]) < 1e-6
    if cb["converged"]:
        assert cb["iterations"] == 41  # the reference's own cfg0 count (tests/golden/cfg0.npz)

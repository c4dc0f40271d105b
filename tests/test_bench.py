"""The bench.py contract on CPU: the reference arm's JSON line (the driver runs it
first, on every N), identical config dicts in both arms, and the launcher's
refusal to report fewer GPUs than asked for."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1604_05872_b200 import fe  # noqa: E402

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"}


def _ref_available():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refkernel as rk

    return rk.available(fe.CONFIGS["c1"], "quad")


def _json_lines(out):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


@pytest.mark.skipif(not _ref_available(), reason="reference sources not emitted (oracle/_ref/src)")
def test_reference_arm_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--configs", "c1,c2", "--steps", "1", "--warmup", "3",
                        "--ref-step-seconds", "0.02"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert KEYS <= set(d)
    assert d["impl"] == "reference" and d["headline"] == "c2" and d["n_gpus"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    # the workload dicts are the ones the GPU arm prints (the driver compares them)
    for name in ("c1", "c2"):
        assert d["configs"][name]["config"] == bench.config_dict(fe.CONFIGS[name], 1, "strong")
    assert d["config"] == bench.config_dict(fe.CONFIGS["c2"], 1, "strong")


@pytest.mark.skipif(not _ref_available(), reason="reference sources not emitted (oracle/_ref/src)")
def test_reference_arm_under_torchrun_prints_once(tmp_path):
    # the driver launches the reference arm like ours: rank 0 alone runs and prints
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr", "127.0.0.1",
                        "--master-port", str(29500 + os.getpid() % 1000),
                        os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--configs", "c1", "--steps", "1", "--warmup", "3",
                        "--ref-step-seconds", "0.02"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2
    assert lines[0]["config"] == bench.config_dict(fe.CONFIGS["c1"], 2, "strong")


def test_refuses_more_gpus_than_visible():
    # no GPU in this container: --gpus 2 must fail loudly, not report a 0/1-GPU run
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--configs", "c1", "--steps", "1"], capture_output=True, text=True,
                       timeout=300)
    import torch

    if torch.cuda.device_count() >= 2:
        pytest.skip("a multi-GPU host")
    assert r.returncode == 2
    assert "CUDA devices" in r.stderr and not _json_lines(r.stdout)


def test_config_dict_and_args():
    a = bench.parse(["--configs", "c3,c1", "--headline", "c5"])
    assert a.configs == ["c3", "c1"] and a.headline == "c1" and a.warmup >= 3
    a = bench.parse([])
    assert a.configs == list(bench.CONFIG_ORDER) and a.headline == "c5"
    assert a.partition == "strong"
    s = bench.config_dict(fe.CONFIGS["c5"], 8, "strong")
    w = bench.config_dict(fe.CONFIGS["c5"], 8, "weak")
    assert s["cells"] == fe.CONFIGS["c5"].ncells and w["cells"] == 8 * fe.CONFIGS["c5"].ncells
    assert "contiguously over 8" in s["parallelism"]


def test_committed_ncu_captures_match_kernel_sources():
    """Every config's committed ncu capture (profiles/ncu_summary.json) belongs to the
    current source of its kernel, so the bench's roofline uses the ncu-counted F_exec
    and DRAM traffic instead of falling back to the flop model."""
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
        summ = json.load(f)
    for cfg in bench.CONFIG_ORDER:
        d = summ[cfg]
        name = d["kernel"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
        assert bench.kernel_source_sha(name) == d["src_sha"], (cfg, name)
        assert bench.ncu_capture(cfg, name) is not None, cfg


def test_kernel_source_sha_ignores_comments(tmp_path, monkeypatch):
    src = tmp_path / "paper_1604_05872_b200" / "csrc"
    src.mkdir(parents=True)
    (src / "pair.cu").write_text("int f() {\n  return 1;  // one\n}\n")
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    a = bench.kernel_source_sha("pair_ws_kernel")
    (src / "pair.cu").write_text("// header\n\nint f() {\n  return 1;  // uno\n}\n")
    assert bench.kernel_source_sha("pair_ws_kernel") == a
    (src / "pair.cu").write_text("int f() {\n  return 2;\n}\n")
    assert bench.kernel_source_sha("pair_ws_kernel") != a

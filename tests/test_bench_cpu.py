"""bench.py host-side pieces (no GPU): both arms quote one workload config, built from the
planner's largest resident batch (827 / 6058 on the B200's reported HBM; a little more here,
where the planner assumes the nominal 183,359 MiB)."""
import argparse

import bench
from paper_2503_09716_b200.configs import get_arch
from paper_2503_09716_b200.engine import resident_plan


def _args(**kw):
    base = dict(prompt_len=512, decode_len=256, batch=None, reserve_gb=14)
    base.update(kw)
    return argparse.Namespace(**base)


def test_workload_config_is_the_planners_resident_batch():
    for name, tag in (("mixtral-8x7b", "BASELINE configs[1]"), ("deepseek-v2-lite", "BASELINE configs[2], 1 GPU")):
        arch = get_arch(name)
        B = resident_plan(arch, 512, 256, reserve_bytes=14 << 30).B
        cfg = bench._workload_config(_args(), arch, 8)
        assert cfg["batch"] == B == cfg["b_a"]
        assert tag in cfg["workload"] and f"B={B} sequences" in cfg["workload"]
        assert cfg["parallelism"] == "replicas x8"


def test_workload_config_batch_cap():
    assert bench._workload_config(_args(batch=64), get_arch("mixtral-8x7b"), 1)["batch"] == 64


def test_measured_reserve_sizes_the_mixtral_batch():
    """Without --reserve-gb the planner keeps the measured per-model reserve (bench.RESERVE_GB):
    Mixtral's 6.25 GiB admits more sequences than the flat 14 GiB; DeepSeek-V2-Lite keeps 14 GiB."""
    mix, ds = get_arch("mixtral-8x7b"), get_arch("deepseek-v2-lite")
    cfg = bench._workload_config(_args(reserve_gb=None), mix, 1)
    assert cfg["hbm_reserve_gb"] == bench.RESERVE_GB["mixtral-8x7b"]
    assert cfg["batch"] == resident_plan(mix, 512, 256, reserve_bytes=int(6.25 * 2**30)).B
    assert cfg["batch"] > resident_plan(mix, 512, 256, reserve_bytes=14 << 30).B
    assert bench._workload_config(_args(reserve_gb=None), ds, 1)["batch"] == \
        resident_plan(ds, 512, 256, reserve_bytes=14 << 30).B

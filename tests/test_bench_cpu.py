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


def test_expert_parallel_plans_fit_the_big_configs():
    """configs[3]/[4] at 8 GPUs: each EP rank holds 1/8 of the routed experts, so the planner sizes B
    next to the rank's own weights (DeepSeek-V2 236B: 445 GB of routed experts, never on one GPU)."""
    from paper_2503_09716_b200.engine import routed_expert_bytes

    hbm = 183_359 << 20
    for name in ("deepseek-v2-236b", "mixtral-8x22b"):
        arch = get_arch(name)
        assert routed_expert_bytes(arch) > hbm
        B8 = resident_plan(arch, 512, 256, reserve_bytes=14 << 30, hbm_bytes=hbm, ep_world=8).B
        B4 = resident_plan(arch, 512, 256, reserve_bytes=14 << 30, hbm_bytes=hbm, ep_world=4).B
        assert B8 > 256 and B8 > B4
    ds = get_arch("deepseek-v2-lite")  # more HBM per rank for KV as the experts spread
    assert resident_plan(ds, 512, 256, reserve_bytes=14 << 30, ep_world=8).B > \
        resident_plan(ds, 512, 256, reserve_bytes=14 << 30).B


def test_use_ep_selection():
    a = _args(ep="auto")
    assert not bench.use_ep(a, get_arch("deepseek-v2-lite"), 1)
    assert bench.use_ep(a, get_arch("deepseek-v2-lite"), 8)
    assert bench.use_ep(a, get_arch("deepseek-v2-236b"), 8)
    assert bench.use_ep(a, get_arch("mixtral-8x22b"), 8)       # 281 GB: experts shard
    assert not bench.use_ep(a, get_arch("mixtral-8x7b"), 8)    # fits one GPU: replicas
    assert bench.use_ep(_args(ep="force"), get_arch("mixtral-8x7b"), 1)
    assert not bench.use_ep(_args(ep="off"), get_arch("deepseek-v2-lite"), 8)

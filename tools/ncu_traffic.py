"""Write profiles/ncu_traffic.json: DRAM read+write bytes per launch of the expert GEMMs at the bench
shapes, from ncu --set full reports of tools/gemm_check.py (same kernels, same per-expert token
counts as the bench configs).  bench.py reports them as roofline.traffic.

  ncu --set full --clock-control none -k regex:moe_gemm -c 2 -o gpurun_out/gemm_mixtral python tools/gemm_check.py mixtral
  ncu --set full --clock-control none -k regex:moe_gemm -c 2 -o gpurun_out/gemm_dsv2 python tools/gemm_check.py dsv2
  ncu --set full --clock-control none -k regex:moe_ffn -c 1 -o gpurun_out/ffn_mixtral_r2b \
      python tools/gemm_prefill_bench.py mixtral-8x7b 227 ffn
  python tools/ncu_traffic.py
"""
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = {"mixtral-8x7b": "gpurun_out/gemm_mixtral.ncu-rep", "deepseek-v2-lite": "gpurun_out/gemm_dsv2.ncu-rep"}
# the fused FFN launch (Mixtral-family default) at the bench's tokens per expert (B = 909: 227)
FFN = {"mixtral-8x7b": ("gpurun_out/ffn_mixtral_r2b.ncu-rep", "tools/gemm_prefill_bench.py mixtral-8x7b 227 ffn")}


def launches(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
        wr = float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
        yield d["Kernel Name"], rd + wr


out = {}
for cfg, rep in CASES.items():
    path = os.path.join(ROOT, rep)
    if not os.path.exists(path):
        continue
    for name, b in launches(path):
        # template argument GATED (first): <1, ...> / <true, ...> is the gate/up GEMM
        targs = name.split("<", 1)[1].split(">", 1)[0] if "<" in name else ""
        key = "gate_up" if targs.split(",")[0].strip() in ("1", "true") else "down"
        out.setdefault(cfg, {})[key] = {"dram_bytes": b, "kernel": name.split("(")[0],
                                        "source": f"ncu --set full of tools/gemm_check.py ({os.path.basename(rep)})"}
for cfg, (rep, cmd) in FFN.items():
    path = os.path.join(ROOT, rep)
    if os.path.exists(path):
        for name, b in launches(path):
            out.setdefault(cfg, {})["ffn"] = {"dram_bytes": b, "kernel": name.split("(")[0],
                                              "source": f"ncu --set full of {cmd} ({os.path.basename(rep)})"}
with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))

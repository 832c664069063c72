"""Per-stage roofline fractions from a bench.py JSON line (profiled eager pass): GEMM stages
against the 3xTF32 tensor peak (algorithmic 2MNK flops), element-wise / epilogue-class stages
against HBM, eigensolver / Cholesky against the FP32 CUDA-core peak.  Stages that overlap
(the side-stream EA) are timed on their own stream.  usage: stage_roofline.py BENCH.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    line = [x for x in open(sys.argv[1]) if x.startswith("{")][-1]
    d = json.loads(line)
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    def num(*keys):
        for k in keys:
            v = pk.get(k)
            if isinstance(v, (int, float)):
                return float(v)
            if isinstance(v, dict) and isinstance(v.get("value"), (int, float)):
                return float(v["value"])
        return None
    bf16 = num("bf16_tflops_sustained", "bf16_dense_tflops_sustained", "bf16_tflops", "bf16_dense_tflops")
    hbm = num("hbm_gbs", "hbm_copy_gbs", "hbm_GBps")
    tf3 = bf16 / 2 / 3 if bf16 else None
    fp32 = 148 * 128 * 2 * 1965e6 / 1e12
    steps = d["steps"]
    rows = ["| stage | ms/step | achieved | peak | fraction |", "|---|---|---|---|---|"]
    for s in d["stages"]:
        ms = s["ms"] / steps
        if ms < 0.02:
            continue
        sec = s["ms"] / 1e3
        name = s["stage"]
        if name.startswith("gemm_") and s["gflop"] > 0 and tf3:
            a = s["gflop"] / sec / 1e3
            rows.append(f"| {name} | {ms:.3f} | {a:.1f} TF/s | {tf3:.0f} TF/s (3xTF32) | {a / tf3:.3f} |")
        elif name.startswith(("ew_", "prec_")) and s["gbytes"] > 0 and hbm:
            a = s["gbytes"] / sec
            rows.append(f"| {name} | {ms:.3f} | {a:.0f} GB/s | {hbm:.0f} GB/s (HBM) | {a / hbm:.3f} |")
        elif name == "eig_sytrd_gt" and hbm:
            a = s["gbytes"] / sec
            rows.append(f"| {name} | {ms:.3f} | {a:.0f} GB/s | {hbm:.0f} GB/s (HBM) | {a / hbm:.3f} |")
        elif s["gflop"] > 0:
            a = s["gflop"] / sec / 1e3
            rows.append(f"| {name} | {ms:.3f} | {a:.2f} TF/s | {fp32:.1f} TF/s (FP32) | {a / fp32:.4f} |")
        else:
            rows.append(f"| {name} | {ms:.3f} | latency-bound | — | — |")
    print("\n".join(rows))


if __name__ == "__main__":
    main()

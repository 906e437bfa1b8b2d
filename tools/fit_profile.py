"""Fit the reference's 4-number device model to the measured B200 per-layer timings of
tools/netbench.py (profiles/r01_netbench.jsonl) and report how well model-only selection
matches measured selection.  usage: python tools/fit_profile.py IN.jsonl OUT.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P  # noqa: E402
from paper_2104_09455_b200 import calibrate  # noqa: E402

rows, per_cfg = [], {}
for line in open(sys.argv[1]):
    d = json.loads(line)
    key = f"{d['net']}/{d['config']}"
    ver = d.get("verify_us", 0.0) / max(1, d["layers"])
    for r in d["per_layer"]:
        lt = calibrate.LayerTiming(P.GemmShape(r["m"], r["n"], r["k"]), r["t_un"] * 1e-6, (r["t_gl"] + ver) * 1e-6,
                                   r["t_one"] * 1e-6)
        rows.append(lt)
        per_cfg.setdefault(key, []).append(lt)
peaks_json = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                         "MEASURED_PEAKS.json")))
peaks = P.DeviceProfile(name="B200", tensor_throughput=peaks_json["bf16_tflops"] * 1e12,
                        alu_throughput=148 * 128 * 2 * peaks_json.get("sm_max_mhz", 1965) * 1e6,
                        memory_bandwidth=peaks_json["hbm_gbs"] * 1e9, verification_launch_latency=0.0)
t0 = time.time()
fit = calibrate.fit_device_profile(rows, P.BINARY16, peaks)
t4 = P.DeviceProfile(name="T4 (reference default)", tensor_throughput=65e12, alu_throughput=8.1e12,
                     memory_bandwidth=320e9, verification_launch_latency=5e-6)
raw = calibrate.evaluate(rows, P.BINARY16, peaks)
ref = calibrate.evaluate(rows, P.BINARY16, t4)


def summary(res):
    return dict(agreement=round(res.agreement, 4),
                model_plan_overhead_pct=round(100 * (res.model_plan_time / res.unprotected_time - 1), 2),
                measured_plan_overhead_pct=round(100 * (res.measured_plan_time / res.unprotected_time - 1), 2))


out = {"source": sys.argv[1], "layers": len(rows), "fit_seconds": round(time.time() - t0, 1),
       "fitted": dict(tensor_tflops=fit.device.tensor_throughput / 1e12, alu_tflops=fit.device.alu_throughput / 1e12,
                      memory_gbs=fit.device.memory_bandwidth / 1e9,
                      verification_latency_us=fit.device.verification_launch_latency * 1e6, **summary(fit)),
       "measured_peaks_unfitted": summary(raw), "t4_reference_default": summary(ref),
       "per_config_fitted": {k: summary(calibrate.evaluate(v, P.BINARY16, fit.device)) for k, v in per_cfg.items()}}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))

"""Times exf_count_transitions and exf_route_replay on 2^21 x 24 traces (E=8, 64)
with CUDA events and checks them against the oracle (diagnostics; the bench
reports the same numbers in its routing_kernels sub-object)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch
    import bench
    peaks = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
    r = bench.measure_routing_kernels(peaks.get("hbm_gbs", 6558.0), torch.cuda.Stream())
    for E, v in r["per_E"].items():
        print(E, {k: (round(x["ms_per_call"] * 1e3, 1), round(x["frac"], 3)) for k, x in v.items()
                  if isinstance(x, dict) and "frac" in x}, "parity", v["parity"],
              "host", v["count_transitions"]["host_entry_ms"], v["route_replay"]["host_entry_ms"],
              "cpu", v["cpu_reference_loops"])

"""Print the last e2e step of gpurun_out/e2e_trace_<workload>.json (GPU activities + host API calls)."""
import json
import re
import sys

wl = sys.argv[1] if len(sys.argv) > 1 else "config2"
show_api = len(sys.argv) > 2
ev = json.load(open(f"gpurun_out/e2e_trace_{wl}.json"))["traceEvents"]
xs = [e for e in ev if e.get("ph") == "X"]
gpu = sorted([e for e in xs if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
fl = [e for e in gpu if "array" in e["name"]]
st = fl[-1]["ts"] + fl[-1]["dur"]
for e in gpu:
    if e["ts"] >= st:
        nm = e["name"]
        m = re.search(r"(\w+_kernel)", nm)
        nm = m.group(1) if m else nm.split("(")[0][-30:]
        print(f"{e['ts'] - st:8.1f} - {e['ts'] + e['dur'] - st:8.1f} ({e['dur']:6.1f}) s{e['args'].get('stream', '?'):<3} {nm} {e['args'].get('bytes', '')}")
if show_api:
    for e in sorted([e for e in xs if e.get("cat") == "cuda_runtime" and e["ts"] >= fl[-1]["ts"]], key=lambda e: e["ts"]):
        print(f"   host {e['ts'] - st:8.1f} +{e['dur']:5.1f} {e['name']}")

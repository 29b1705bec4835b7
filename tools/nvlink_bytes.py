"""NVLink data counters around a command: total Tx / Rx bytes per GPU (nvidia-smi nvlink -gt d).

    python tools/nvlink_bytes.py OUT_JSON -- <command ...>

Reads the per-link data-throughput counters of every visible GPU before and after the
command and writes the per-GPU byte deltas plus the command's wall time."""
import json
import re
import subprocess
import sys
import time


def counters():
    out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d"], capture_output=True, text=True).stdout
    gpu, res = None, {}
    for line in out.splitlines():
        m = re.match(r"GPU (\d+):", line)
        if m:
            gpu = int(m.group(1))
            res[gpu] = {"tx": 0, "rx": 0}
            continue
        m = re.search(r"Link \d+: Data (Tx|Rx): (\d+) KiB", line)
        if m and gpu is not None:
            res[gpu][m.group(1).lower()] += int(m.group(2)) * 1024
    return res, out


out_path = sys.argv[1]
cmd = sys.argv[sys.argv.index("--") + 1:]
before, raw_before = counters()
t0 = time.time()
rc = subprocess.run(cmd).returncode
wall = time.time() - t0
after, raw_after = counters()
delta = {g: {k: after[g][k] - before[g].get(k, 0) for k in ("tx", "rx")} for g in after}
json.dump({"cmd": " ".join(cmd), "rc": rc, "wall_s": wall, "bytes": delta,
           "raw_sample": raw_after.splitlines()[:12]}, open(out_path, "w"), indent=1)
print(json.dumps({"rc": rc, "wall_s": round(wall, 1),
                  "tx_GB": {g: round(v["tx"] / 1e9, 2) for g, v in delta.items()}}))

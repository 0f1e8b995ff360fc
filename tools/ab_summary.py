"""Summarise tools/gpu_env_ab.sh / gpu_geglu_ab.sh logs: mean config-3 ms per arm and width."""
import re
import sys

cur, res = None, {}
for line in open(sys.argv[1]):
    if re.match(r"^(on|off|fused|unfused):", line):
        cur = line.split(":")[0]
    elif line.startswith("{") and cur:
        m = re.search(r'"bits": (\d).*"ms": ([\d.]+)', line)
        res.setdefault((cur, m.group(1)), []).append(float(m.group(2)))
    elif "passed" in line or "failed" in line:
        print(line.strip())
for k, v in sorted(res.items()):
    print(k, [round(x, 2) for x in v], round(sum(v) / len(v), 2))

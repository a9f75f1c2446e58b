"""Per-kernel launch counts / time shares of an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_shares.py gpurun_out/x_launches.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit() and r[12] == "gpu__time_duration.sum"]
tot = collections.Counter()
cnt = collections.Counter()
for r in rows:
    name = r[4].split("(")[0][:70]
    tot[name] += float(r[14].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}[r[13]]
    cnt[name] += 1
all_ms = sum(tot.values())
for name, ms in tot.most_common():
    print(f"{name:70s} launches {cnt[name]:4d}  total {ms:9.3f} ms  mean {ms / cnt[name] * 1e3:9.2f} us  share {100 * ms / all_ms:5.1f}%")

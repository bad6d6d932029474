"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``): share of
serialised kernel time per kernel, and the share of liblms's own kernels.

Usage: python scripts/launch_summary.py gpurun_out/ev_launches.csv [--skip-until zvc_]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    skip = sys.argv[3] if len(sys.argv) > 3 and sys.argv[2] == "--skip-until" else None
    rows = list(csv.reader(open(path)))
    hdr, tot, cnt = None, collections.Counter(), collections.Counter()
    started = skip is None
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        if not started:
            if skip not in name:
                continue
            started = True
        tot[name] += float(d["Metric Value"])
        cnt[name] += 1
    all_ns = sum(tot.values())
    ours = {k: v for k, v in tot.items() if "lms::" in k}
    print(f"launches {sum(cnt.values())}, serialised kernel time {all_ns / 1e6:.1f} ms"
          + (f" (from the first launch matching {skip!r})" if skip else ""))
    print(f"liblms kernels: {sum(cnt[k] for k in ours)} launches, {sum(ours.values()) / max(all_ns, 1) * 100:.1f} %"
          " of serialised kernel time")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:20]:
        print(f"{v / all_ns * 100:6.2f} %  {cnt[k]:6d}  {k[:110]}")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Turns ncu output into the text tables kept under profiles/.

  ncu_tables.py launches <launches.csv>           per-launch list + per-kernel totals (ncu --metrics ... --csv --log-file)
  ncu_tables.py raw <report.ncu-rep> [regex ...]  selected metrics of every captured launch (ncu --set full)
  ncu_tables.py traffic <launches.csv> <config> <hash> <max_cost> [profiles/roofline_traffic.json]
                                                  the entry bench.py reads for exactly that workload (printed; merged into
                                                  the JSON file when one is named)
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short(name: str) -> str:
    name = re.sub(r"^void\s+", "", name.split("(")[0] if not name.startswith("void") else name[5:].split("(")[0] + "")
    return re.sub(r"\(int\)", "", name).strip()


def read_launches(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    d = collections.OrderedDict()
    for x in csv.DictReader(lines):
        e = d.setdefault(int(x["ID"]), {"name": short(x["Kernel Name"])})
        v, u, m = float(x["Metric Value"].replace(",", "")), x["Metric Unit"], x["Metric Name"]
        if m == "gpu__time_duration.sum":
            e["ms"] = v * SCALE[u]
        elif m.startswith("dram__bytes"):
            e["rd" if "read" in m else "wr"] = v * BYTES[u]
        elif m.startswith("lts__t_sector_hit_rate"):
            e["l2hit"] = v
        elif m.startswith("l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom"):
            e["atom"] = v
        elif m == "smsp__inst_executed.sum":
            e["inst"] = v
    return d


def launches(path):
    d = read_launches(path)
    print(f"{'id':>4s} {'kernel':28s} {'ms':>9s} {'warp-inst':>14s} {'dram rd GB':>11s} {'dram wr GB':>11s} {'L2 hit %':>9s} {'atomics':>10s}")
    tot = collections.OrderedDict()
    for k, e in d.items():
        print(f"{k:4d} {e['name']:28s} {e['ms']:9.4f} {int(e.get('inst', 0)):14d} {e.get('rd', 0) / 1e9:11.4f} {e.get('wr', 0) / 1e9:11.4f}"
              f" {e.get('l2hit', float('nan')):9.1f} {int(e.get('atom', 0)):10d}")
        t = tot.setdefault(e["name"], [0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0])
        for i, v in enumerate((1, e["ms"], e.get("inst", 0), e.get("rd", 0), e.get("wr", 0), e.get("atom", 0),
                               e.get("l2hit", 0.0) * e["ms"])):
            t[i] += v
    all_ms = sum(t[1] for t in tot.values())
    print(f"\n{'kernel':28s} {'launches':>8s} {'ms':>9s} {'share':>7s} {'warp-inst':>14s} {'dram rd GB':>11s} {'dram wr GB':>11s} {'L2 hit %':>9s} {'atomics':>10s}")
    for n, t in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:28s} {t[0]:8d} {t[1]:9.3f} {100 * t[1] / all_ms:6.1f}% {int(t[2]):14d} {t[3] / 1e9:11.3f} {t[4] / 1e9:11.3f}"
              f" {t[6] / max(t[1], 1e-9):9.1f} {int(t[5]):10d}")
    print(f"total {all_ms:.3f} ms  (cold-cache, serialised launches: compare shares, not absolutes)")


def traffic(path, config, hash_name, max_cost, merge_into=None, source=None):
    import os

    d = read_launches(path)
    def rewrite(name):  # k_screen<W, 2, PAIR> is the tile-shaped phase B (KIND_REWRITE), not screening
        m = re.match(r"k_screen<\s*\d+,\s*(\d+)", name)
        return bool(m) and m.group(1) == "2"

    scr = [e for e in d.values() if e["name"].startswith("k_screen") and not rewrite(e["name"])]
    mat = [e for e in d.values() if e["name"].startswith("k_materialize") or rewrite(e["name"])]
    small = [e for e in d.values() if e["name"].startswith("k_level")]
    scr_ms = sum(e["ms"] for e in scr)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2402_12373_b200 import build as B

    entry = {
        "source": source or f"{path} (ncu metrics pass over one learn() of the workload)",
        "build_digest": B._sources_digest()[:16],
        "k_screen_launches": len(scr),
        "k_screen_ms_under_ncu": scr_ms,
        "k_screen_dram_bytes_per_launch": sum(e["rd"] + e["wr"] for e in scr) / max(len(scr), 1),
        "k_screen_dram_bytes_per_step": sum(e["rd"] + e["wr"] for e in scr),
        "k_screen_warp_instructions_per_step": sum(e["inst"] for e in scr),
        "k_screen_l2_hit_pct": sum(e.get("l2hit", 0.0) * e["ms"] for e in scr) / max(scr_ms, 1e-9),
        "k_screen_atom_ops_per_step": sum(e.get("atom", 0) for e in scr),
        "k_materialize_dram_bytes_per_step": sum(e["rd"] + e["wr"] for e in mat),
        "k_materialize_warp_instructions_per_step": sum(e["inst"] for e in mat),
        "k_level_small_launches": len(small),
        "all_kernels_ms_under_ncu": sum(e["ms"] for e in d.values()),
    }
    key = f"{config}|{hash_name}|{max_cost}"
    print(json.dumps({key: entry}, indent=1))
    if merge_into:
        try:
            with open(merge_into) as fh:
                prof = json.load(fh)
        except Exception:
            prof = {}
        if "entries" not in prof:
            prof = {"entries": {}}
        prof["entries"][key] = entry
        with open(merge_into, "w") as fh:
            json.dump(prof, fh, indent=1, sort_keys=True)


DEFAULT = [r"^gpu__time_duration\.sum$", r"^launch__grid_size$", r"^launch__registers_per_thread$",
           r"^launch__occupancy_limit_(registers|shared_mem)$", r"^smsp__inst_executed\.sum$",
           r"^smsp__issue_active\.avg\.pct_of_peak_sustained_active$",
           r"^sm__inst_executed_pipe_(alu|fma|lsu)\.avg\.pct_of_peak_sustained_active$",
           r"^sm__pipe_(fmaheavy|alu)_cycles_active\.avg\.pct_of_peak_sustained_elapsed$",
           r"^sm__warps_active\.avg\.pct_of_peak_sustained_active$", r"^dram__bytes_(read|write)\.sum$",
           r"^gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed$", r"^dram__throughput\.avg\.pct_of_peak_sustained_elapsed$",
           r"^lts__t_sector_hit_rate\.pct$", r"^l1tex__t_sector_hit_rate\.pct$",
           r"^l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom\.sum$", r"^lts__t_sectors_op_atom\.sum$", r"^lts__t_sectors_op_red\.sum$",
           r"^smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio$"]


def raw(path, pats):
    if path.endswith(".csv"):  # the raw page exported on the GPU box (`ncu -i rep --page raw --csv`)
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    pats = [re.compile(p) for p in (pats or DEFAULT)]
    kn = hdr.index("Kernel Name")
    print("launch: " + "  ".join(f"#{i}={short(r[kn])}" for i, r in enumerate(data)))
    print(f"{'metric':88s}" + "".join(f"{'#' + str(i):>14s}" for i in range(len(data))))
    for j, h in enumerate(hdr):
        if not any(p.search(h) for p in pats):
            continue
        vals = []
        for r in data:
            try:
                vals.append(f"{float(r[j].replace(',', '')):14.3f}")
            except ValueError:
                vals.append(f"{r[j]:>14s}")
        if "issue_stalled" in h and all(float(v) < 0.05 for v in vals):
            continue
        print(f"{h:88s}" + "".join(vals) + f" {units[j]}")


if __name__ == "__main__":
    cmd = sys.argv[1]
    {"launches": lambda: launches(sys.argv[2]),
     "traffic": lambda: traffic(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5], sys.argv[6] if len(sys.argv) > 6 else None),
     "raw": lambda: raw(sys.argv[2], sys.argv[3:])}[cmd]()

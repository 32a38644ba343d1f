#!/usr/bin/env python3
"""Summarise an `ncu --set full` report of the test kernels into profiles/ JSON.

    python tools/ncu_summary.py gpurun_out/full_r01.ncu-rep --label "..." \
        --names voronoi,sign_of_offset,ray_crossing --points 2147483648 \
        --out profiles/ncu_full_r01_c5.json [--traffic profiles/traffic_r01.json --key c5]

Per kernel: duration, DRAM bytes, issue / pipe utilisation, warps, registers,
L1/L2 figures; the SASS instruction mix (executed warp instructions per
opcode, from the source page) and the warp-stall breakdown. With --traffic the
per-launch DRAM bytes are also written where bench.py reads them
(roofline.traffic).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def ncu(rep: str, *args: str) -> str:
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True,
                          check=True).stdout


def raw_rows(rep: str):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def to_bytes(value: str, unit: str) -> float:
    return float(value.replace(",", "")) * UNIT.get(unit, 1)


def source_blocks(rep: str):
    """Yield (kernel name, header, rows) from the SASS source page."""
    text = ncu(rep, "--page", "source", "--csv", "--print-source", "sass")
    name, hdr, rows = None, None, []
    for r in csv.reader(io.StringIO(text)):
        if not r:
            continue
        if r[0] == "Kernel Name":
            if name is not None:
                yield name, hdr, rows
            name, hdr, rows = r[1], None, []
        elif hdr is None:
            hdr = r
        else:
            rows.append(r)
    if name is not None:
        yield name, hdr, rows


def mix_and_stalls(hdr, rows):
    ie = hdr.index("Instructions Executed")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    mix, stalls = collections.Counter(), collections.Counter()
    for r in rows:
        t = r[1].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        mix[op] += int(r[ie] or 0)
        for i in stall_cols:
            stalls[hdr[i]] += int(r[i] or 0)
    total = sum(mix.values())
    s_total = sum(stalls.values()) or 1
    return ({op: n for op, n in mix.most_common(20)}, total,
            {k: round(v / s_total * 100, 1) for k, v in stalls.most_common(10)})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--label", required=True)
    ap.add_argument("--names", required=True, help="comma-separated, one per profiled launch")
    ap.add_argument("--points", type=int, required=True)
    ap.add_argument("--bytes-per-point", type=float, default=8.125)
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic")
    ap.add_argument("--key")
    ap.add_argument("--merge", action="store_true",
                    help="add these kernels to an existing --out file instead of replacing it")
    a = ap.parse_args()
    names = a.names.split(",")
    hdr, units, data = raw_rows(a.rep)
    if len(data) != len(names):
        raise SystemExit(f"{len(data)} launches in the report, {len(names)} names")
    out = {"capture": a.label, "kernels": {}}
    # the source page lists every profiled launch twice (two views); keep one
    blocks = list(source_blocks(a.rep))
    if len(blocks) == 2 * len(names):
        blocks = blocks[0::2]
    for name, row, (kname, shdr, srows) in zip(names, data, blocks):
        k = {}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                k[m] = f"{row[i]} {units[i]}".strip()
        rd = to_bytes(row[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(row[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        k["dram_bytes_per_launch"] = rd + wr
        k["algorithmic_bytes_per_launch"] = a.bytes_per_point * a.points
        mix, total, stalls = mix_and_stalls(shdr, srows)
        k["sass_kernel"] = kname
        # executed warp instructions x 32 lanes per test (point or pair)
        k["thread_instructions_per_test"] = round(32 * total / a.points, 2)
        k["instruction_mix"] = mix
        k["warp_stall_pct"] = stalls
        out["kernels"][name] = k
    if a.merge and Path(a.out).exists():
        prev = json.loads(Path(a.out).read_text())
        prev["kernels"].update(out["kernels"])
        prev["capture"] = prev["capture"] + " | " + a.label
        out = prev
    Path(a.out).write_text(json.dumps(out, indent=1) + "\n")
    print(f"wrote {a.out}")
    if a.traffic:
        p = Path(a.traffic)
        tj = json.loads(p.read_text()) if p.exists() else {}
        ent = tj.get(a.key, {}) if a.merge else {}
        ent["points"] = a.points
        ent.setdefault("dram_bytes_per_launch", {}).update(
            {n: out["kernels"][n]["dram_bytes_per_launch"] for n in names})
        tj[a.key] = ent
        p.write_text(json.dumps(tj, indent=1) + "\n")
        print(f"updated {p} [{a.key}]")


if __name__ == "__main__":
    main()

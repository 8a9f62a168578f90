"""Basic-block breakdown of one kernel from an ncu --set full --import-source
capture: instructions executed and warp stall samples per run of SASS
instructions with equal execution counts (tools/ only).
    python tools/ncu_blocks.py report.ncu-rep [top]   (JSON to stdout)"""
import collections
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kernel, hdr, ins = rows[0][1], rows[1], []
ia, isrc = hdr.index("Address"), hdr.index("Source")
ie, iss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = None
for r in rows[2:]:
    if not r or not r[0].startswith("0x"):
        if r and r[0] == "Kernel Name":
            break  # first kernel of the report only
        continue
    a = int(r[ia], 16)
    base = a if base is None else base
    src = r[isrc].strip()
    op = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0]
    ins.append((a - base, op, int(r[ie]), int(r[iss])))
tot, tots = sum(x[2] for x in ins), sum(x[3] for x in ins)
blocks, cur = [], None
for off, op, e, s in ins:
    if cur and cur["exec"] == e:
        cur["n"] += 1
        cur["samples"] += s
        cur["end"] = off
        cur["ops"][op] += 1
    else:
        cur = {"start": off, "end": off, "exec": e, "n": 1, "samples": s, "ops": collections.Counter({op: 1})}
        blocks.append(cur)
blocks.sort(key=lambda b: -b["exec"] * b["n"])
print(json.dumps({
    "kernel": kernel, "inst_executed": tot, "stall_samples": tots,
    "blocks": [{"sass_offsets": [hex(b["start"]), hex(b["end"])], "instructions": b["n"],
                "executions": b["exec"], "inst_share": round(b["exec"] * b["n"] / tot, 4),
                "stall_share": round(b["samples"] / max(tots, 1), 4),
                "top_ops": dict(b["ops"].most_common(4))} for b in blocks[:top]]}, indent=1))

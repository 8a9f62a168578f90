"""Summarise an ncu --set full report: per kernel launch, duration, issue,
occupancy, pipes, DRAM bytes and the top stall reasons.

    python tools/ncu_summary.py report.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ns": "gpu__time_duration.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "ipc_active": "sm__inst_executed.avg.per_cycle_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "sm_clock_hz": "smsp__cycles_elapsed.avg.per_second",
}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        ent = {"kernel": d.get("Kernel Name", ""), "id": d.get("ID")}
        for k, m in KEYS.items():
            v = d.get(m)
            try:
                v = float(v.replace(",", ""))
            except Exception:  # noqa: BLE001
                pass
            unit = u.get(m, "")
            if isinstance(v, float) and k.startswith("dram") and unit:
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            if isinstance(v, float) and k == "duration_ns" and unit:
                v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
            ent[k] = v
        st = []
        for m, v in d.items():
            if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(v), m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except Exception:  # noqa: BLE001
                    pass
        ent["stalls"] = {n: round(v, 3) for v, n in sorted(st, reverse=True)[:6]}
        res.append(ent)
    return res


if __name__ == "__main__":
    res = load(sys.argv[1])
    for e in res:
        print(json.dumps(e))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)

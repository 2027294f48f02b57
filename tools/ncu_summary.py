"""Summarise an ncu report: key raw metrics, stall reasons, top instructions,
opcode histogram per kernel.   python tools/ncu_summary.py report.ncu-rep"""

import csv
import io
import subprocess
import sys
from collections import Counter

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__ops_path_tensor_src_fp64.sum", "sm__warps_active.avg.per_cycle_active",
       "launch__registers_per_thread", "launch__occupancy_limit_registers",
       "launch__occupancy_limit_shared_mem", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
       "smsp__inst_executed.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print("==", r[ix["Kernel Name"]][:80])
        for k in RAW:
            if k in ix:
                print(f"   {k:80s} {r[ix[k]]} {units[ix[k]]}")
    src = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv"]))))
    blocks, cur = [], None
    for r in src:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r:
            cur["rows"].append(r)
    seen = set()
    for b in blocks:
        if b["name"] in seen or "hdr" not in b:
            continue
        seen.add(b["name"])
        h = b["hdr"]
        ix = {k: i for i, k in enumerate(h)}
        samp = "Warp Stall Sampling (All Samples)"
        tot = sum(int(r[ix[samp]] or 0) for r in b["rows"])
        print("==", b["name"][:80], "stall samples", tot)
        reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
        agg = {k: sum(int(r[ix[k]] or 0) for r in b["rows"]) for k in reasons}
        print("   stalls:", ", ".join(f"{k[6:]}={v / max(tot, 1):.2f}"
                                      for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
        c = Counter()
        for r in b["rows"]:
            toks = r[ix["Source"]].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            c[op.split(".")[0]] += int(r[ix["Instructions Executed"]] or 0)
        dmma = c.get("DMMA", 0)
        total = sum(c.values())
        print(f"   instructions/DMMA {total / max(dmma, 1):.2f};",
              ", ".join(f"{k}={v / max(dmma, 1):.2f}" for k, v in c.most_common(14)))
        top = sorted(b["rows"], key=lambda r: -int(r[ix[samp]] or 0))[:12]
        for r in top:
            print(f"   {int(r[ix[samp]]) / max(tot, 1):6.3f}  {r[ix['Source']][:70]}")


if __name__ == "__main__":
    main()

"""Stall reasons per code region of the warp-specialized engine (producer vs
consumer), split at the setmaxnreg instructions.  python tools/ncu_regions.py rep"""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; data = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r; continue
    if hdr and r and len(r) == len(hdr): data.append(r)
ix = {k: i for i, k in enumerate(hdr)}
samp = "Warp Stall Sampling (All Samples)"
reasons = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
region = "prologue"; agg = {}
for r in data:
    src = r[ix["Source"]]
    if "USETMAXREG.DEALLOC" in src: region = "producer"
    if "USETMAXREG.ALLOC" in src or "USETMAXREG.TRY_ALLOC" in src: region = "consumer"
    a = agg.setdefault(region, {"samples": 0, "inst": 0, "dmma": 0, **{k: 0 for k in reasons}})
    a["samples"] += int(r[ix[samp]] or 0)
    ie = int(r[ix["Instructions Executed"]] or 0)
    a["inst"] += ie
    if "DMMA" in src: a["dmma"] += ie
    for k in reasons: a[k] += int(r[ix[k]] or 0)
tot = sum(a["samples"] for a in agg.values())
for reg, a in agg.items():
    top = sorted(((a[k], k) for k in reasons), reverse=True)[:7]
    print(f"{reg:9s} samples {a['samples'] / tot:.2f} inst {a['inst']:.3e} dmma {a['dmma']:.3e}: " +
          ", ".join(f"{k[6:]}={v / max(a['samples'], 1):.2f}" for v, k in top))

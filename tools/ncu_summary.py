"""Fold the per-kernel exports of tools/gpu_ncu_all.sh (TAG_<kernel>.raw.csv + .lines.txt under
gpurun_out/) into one JSON for profiles/:  python tools/ncu_summary.py TAG OUT.json"""
import csv, glob, json, os, sys
tag, out = sys.argv[1], sys.argv[2]
res = {"source": "ncu --set full --import-source on --clock-control none, one launch per kernel inside a CH mp_orth "
                 "solve (tools/gpu_ncu_all.sh; .ncu-rep files exported on the box and deleted); per-source-line hot "
                 "spots from tools/sass_lines.py", "kernels": {}}
for f in sorted(glob.glob(f"gpurun_out/{tag}_*.raw.csv")):
    k = os.path.basename(f)[len(tag) + 1:-len(".raw.csv")]
    rows = [r for r in csv.reader(l for l in open(f) if not l.startswith("=="))]
    if len(rows) < 3:
        continue
    h, u, v = rows[0], rows[1], rows[2]
    d = {}
    for i, name in enumerate(h):
        if "__" in name and i < len(v):
            d[name] = f"{v[i]} {u[i]}".strip()
    if "Kernel Name" in h:
        d["kernel_name"] = v[h.index("Kernel Name")]
    lf = f[:-len(".raw.csv")] + ".lines.txt"
    if os.path.exists(lf):
        d["hot_source_lines"] = [l.strip() for l in open(lf) if " instr " in l][:12]
    res["kernels"][k] = d
json.dump(res, open(out, "w"), indent=1)
print(out, list(res["kernels"]))

"""Map an ncu SASS source page to CUDA source lines (needs -lineinfo):
   python tools/sass_lines.py REPORT.ncu-rep KERNEL_SUBSTRING CUBIN [top]
Aggregates 'Instructions Executed' and warp-stall samples per source line, using the
offsets of nvdisasm -g on the cubin (the report's SASS addresses are absolute; the kernel's
first instruction is offset 0)."""
import collections, csv, io, re, subprocess, sys

rep, ksub, cubin = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{ksub}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
name = rows[0][1]
h = rows[1]
ia, isrc, iex, isamp = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index(
    "Warp Stall Sampling (All Samples)")
recs = []
for r in rows[2:]:
    if len(r) <= isamp or not r[ia].startswith("0x"):
        break
    recs.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[isamp] or 0)))
base = recs[0][0]
# mangled name: find in cubin symbol list the function whose SASS length matches
syms = subprocess.run(["cuobjdump", "-symbols", cubin], capture_output=True, text=True).stdout
cands = [l.split()[-1] for l in syms.splitlines() if "STT_FUNC" in l and "STO_ENTRY" in l]
want = re.sub(r"\W", "", ksub)
mangled = None
for c in cands:
    dem = subprocess.run(["cu++filt", c], capture_output=True, text=True).stdout.strip()
    if dem.replace(" ", "").startswith(name.replace(" ", "")[:60]) or (want in c and mangled is None):
        mangled = c
        if dem.replace(" ", "").startswith(name.replace(" ", "")[:60]):
            break
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
sec = dis.split(f".text.{mangled}:", 1)[1]
sec = re.split(r"\n\s*\.section\s", sec, maxsplit=1)[0]
line_of = {}
cur = None
for l in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0, 0])
ti = ts = 0
for a, s, n, smp in recs:
    key = line_of.get(a - base, ("?", 0))
    agg[key][0] += n
    agg[key][1] += smp
    ti += n
    ts += smp
print(f"{name}\n{mangled}\ninstructions {ti}  samples {ts}")
for (f, ln), (n, smp) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{f}:{ln:5d}  instr {n:10d} ({100*n/max(ti,1):5.1f}%)  samples {smp:6d} ({100*smp/max(ts,1):5.1f}%)")

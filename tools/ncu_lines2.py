"""Per-source-line instructions and stall samples of one kernel in an ncu
report (ncu --page source).  ncu can label lines of one header with the
name of another when several are compiled together: --remap A=B shows
lines labelled A with B's source text."""
import argparse, collections, csv, os, subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("kernel")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--remap", action="append", default=[])
ap.add_argument("--src", default=os.path.join(os.path.dirname(__file__), "..", "paper_2009_07785_b200", "csrc"))
a = ap.parse_args()
remap = dict(x.split("=") for x in a.remap)
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + a.kernel], capture_output=True, text=True).stdout
ie = collections.Counter(); st = collections.Counter(); lsb = collections.Counter()
f = None; cur = None; hdr = None
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        f = os.path.basename(r[1]); f = remap.get(f, f); continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not hdr or len(r) < 8:
        continue
    if r[0] != "":
        cur = (f, int(r[0])); continue
    try:
        ie[cur] += float(r[hdr.index("Instructions Executed")] or 0)
        st[cur] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        lsb[cur] += float(r[hdr.index("stall_long_sb")] or 0)
    except (ValueError, IndexError):
        pass
T = sum(ie.values()) or 1; S = sum(st.values()) or 1
print(f"total warp instructions {T:.0f}, stall samples {S:.0f}")
texts = {}
def text(k):
    p = os.path.join(a.src, k[0])
    if p not in texts:
        texts[p] = open(p).read().splitlines() if os.path.exists(p) else []
    L = texts[p]
    return L[k[1] - 1].strip()[:80] if 0 < k[1] <= len(L) else ""
keys = sorted(set(ie) | set(st), key=lambda k: -(ie[k] / T + st[k] / S))
for k in keys[:a.top]:
    print(f"{ie[k]/T*100:5.1f}% inst {st[k]/S*100:5.1f}% stall ({lsb[k]/S*100:4.1f}% lsb) {k[0]}:{k[1]} {text(k)}")

"""Per source line of one kernel: L1 tag requests (global), L1 shared wavefronts, L2 sectors (tools helper)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
hdr, f, agg = None, "", {}
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif len(r) > 6 and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[2] == "-":
        def v(name):
            try:
                return float(r[hdr.index(name)] or 0)
            except (ValueError, IndexError):
                return 0.0
        agg[f"{f}:{r[0]}"] = (v("L1 Tag Requests Global"), v("L1 Wavefronts Shared"), v("L2 Theoretical Sectors Global"),
                              r[1].strip()[:60])
tot = [sum(x[i] for x in agg.values()) for i in range(3)]
print("totals: L1 tag req global %.3g, L1 wavefronts shared %.3g, L2 sectors global %.3g" % tuple(tot))
for k, x in sorted(agg.items(), key=lambda kv: -(kv[1][0] + kv[1][1]))[:top]:
    print(f"{k:20s} tagreq {x[0]:10.3g} smem_wf {x[1]:10.3g} l2sect {x[2]:10.3g}  {x[3]}")

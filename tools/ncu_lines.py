"""Aggregate ncu source-page samples per CUDA source line (tools helper, not product)."""
import csv, sys, subprocess
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
file = None; agg = {}; tot = 0; instr = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        file = r[1].split("/")[-1]; continue
    if len(r) > 6 and r[0] not in ("Line No",) and r[2] == "-":
        try:
            s = float(r[4]); ie = float(r[7])
        except ValueError:
            continue
        key = f"{file}:{r[0]}"
        agg[key] = (agg.get(key, (0, 0, ""))[0] + s, agg.get(key, (0, 0, ""))[1] + ie, r[1].strip()[:90])
        tot += s
print("total samples", tot)
for k, (s, ie, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*s/tot:5.1f}%  inst {ie:10.0f}  {k:22s} {src}")

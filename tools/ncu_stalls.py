"""Top source lines of one kernel by warp-stall samples, with the dominant stall reasons (tools helper)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
hdr, res, f = None, [], ""
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif len(r) > 6 and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[2] == "-":
        try:
            s = float(r[4])
        except ValueError:
            continue
        st = {h[6:]: float(r[i]) for i, h in enumerate(hdr)
              if h.startswith("stall_") and "Not" not in h and r[i] not in ("", "-") and float(r[i]) > 0.1 * s}
        res.append((s, f"{f}:{r[0]}", r[1].strip()[:70], st))
tot = sum(x[0] for x in res)
for s, k, src, st in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100 * s / tot:5.1f}% {k:18s} {src:70s} {st}")

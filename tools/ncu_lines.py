"""Aggregate ncu source-page stall samples per CUDA source line (dev tool).

usage: ncu -i rep --page source --csv --print-source cuda,sass > s.csv
       python tools/ncu_lines.py s.csv [top]"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    cur_file, hdr, out = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            ix = {n: i for i, n in enumerate(r)}
            continue
        if hdr is None or r[0] in ("Function Name",):
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        def g(name):
            v = r[ix[name]] if ix.get(name) is not None and ix[name] < len(r) else ""
            try:
                return int(float(v or 0))
            except ValueError:
                return 0
        out.append((g("Warp Stall Sampling (All Samples)"), g("Instructions Executed"), cur_file,
                    line, r[1].strip()[:90]))
    tot = sum(o[0] for o in out)
    print(f"total samples {tot}")
    for smp, ex, f, ln, src in sorted(out, key=lambda o: -o[0])[:top]:
        print(f"{smp:6d} {100.0 * smp / max(tot, 1):5.1f}% {ex:10d}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()

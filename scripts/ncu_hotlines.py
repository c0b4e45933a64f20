"""Top source lines by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows, fname, hdr = [], None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]; continue
    if r[0] in ('Function Name',):
        continue
    if r[0] == 'Line No':
        hdr = r; continue
    if hdr and fname and r[0].isdigit() and r[2] == '-':
        try:
            rows.append((int(r[4]), int(r[5]), fname, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in rows)
print("total samples", tot)
for s, ni, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {ni:7d} {f}:{ln:<5d} {src}")

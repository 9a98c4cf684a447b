"""Per-source-line hot spots of an .ncu-rep (needs -lineinfo and
--import-source on): warp-stall samples and instructions executed per CUDA
line, top N by samples. Usage: python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv
import subprocess
import sys


def main(path, top=30):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    fname, rows, hdr = '?', [], None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == 'File Path':
            fname = r[1].rsplit('/', 1)[-1]
        elif r[0] == 'Line No':
            hdr = r
        elif hdr and r[0].isdigit() and len(r) == len(hdr):
            try:
                samp, inst = int(r[4]), int(r[7])
            except ValueError:
                continue
            rows.append((samp, inst, fname, int(r[0]), r[1].strip()[:90],
                         {h: r[i] for i, h in enumerate(hdr) if h.startswith('stall_') and '(' not in h}))
    tot = sum(x[0] for x in rows) or 1
    for samp, inst, f, ln, src, st in sorted(rows, reverse=True)[:top]:
        big = sorted(((int(v), k[6:]) for k, v in st.items() if v.isdigit()), reverse=True)[:3]
        print(f"{100 * samp / tot:5.1f}% {inst:>11} {f}:{ln:<5} {src}  [{', '.join(f'{k}={v}' for v, k in big)}]")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

"""Summarise TLRB_TRACE stderr lines: total qrcp / jacobi / panel ms."""
import re
import sys

q = j = pnl = 0.0
nbat = 0
for ln in open(sys.argv[1]):
    m = re.search(r"qrcp ([\d.]+) ms\s+jacobi ([\d.]+) ms", ln)
    if m:
        q += float(m.group(1)); j += float(m.group(2)); nbat += 1
    m = re.search(r"potrf\+trsm\+syrk ([\d.]+) ms", ln)
    if m:
        pnl += float(m.group(1))
print(f"batches {nbat}  qrcp(+M formation) {q:.0f} ms  jacobi(+final GEMM) {j:.0f} ms  panel {pnl:.0f} ms")

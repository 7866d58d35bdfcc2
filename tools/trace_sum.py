"""Summarise TLRB_TRACE stderr lines: total qrcp / jacobi / panel /
factored-QR / apply-Q ms.   python tools/trace_sum.py trace.log"""
import re
import sys

tot = {"qrcp": 0.0, "jacobi": 0.0, "panel": 0.0, "factored-QR": 0.0, "apply-Q": 0.0}
nbat = 0
for ln in open(sys.argv[1]):
    m = re.search(r"qrcp ([\d.]+) ms\s+jacobi ([\d.]+) ms", ln)
    if m:
        tot["qrcp"] += float(m.group(1)); tot["jacobi"] += float(m.group(2)); nbat += 1
    m = re.search(r"potrf\+trsm\+syrk ([\d.]+) ms", ln)
    if m:
        tot["panel"] += float(m.group(1))
    m = re.search(r"(factored-QR|apply-Q) \d+ factors ([\d.]+) ms", ln)
    if m:
        tot[m.group(1)] += float(m.group(2))
print(f"batches {nbat}  " + "  ".join(f"{k} {v:.0f} ms" for k, v in tot.items()))

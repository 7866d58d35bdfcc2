mkdir -p gpurun_out
out=gpurun_out/r02_sweep.jsonl; : > $out
for q in 0 1; do for r in 0.45 0.35 0.3 0.25 0.2; do
  TLRB_DENSE_BY_QRCP=$q TLRB_DENSE_FRAC=$r timeout 300 python tools/c3_once.py >> $out 2>> gpurun_out/r02_sweep.err
done; done
python tools/c3_once.py C2 >> $out 2>> gpurun_out/r02_sweep.err
cat $out

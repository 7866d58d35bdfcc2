mkdir -p gpurun_out
out=gpurun_out/r02_sweep_final2.jsonl; : > $out
for r in 0.12 0.08 0.05 0.03; do
  TLRB_DENSE_FRAC=$r timeout 300 python tools/c3_once.py >> $out 2>> gpurun_out/r02_sweep_final.err
done
cat $out | cut -c1-330

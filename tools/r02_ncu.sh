# ncu evidence at C3 (one evaluation through tools/trace_cfg.py), after a
# clean run of the same command.  Outputs under gpurun_out/.
CMD="python tools/trace_cfg.py C3 --no-warm"
$CMD > gpurun_out/r02_ncu_plain.out 2>&1 || exit 1
# launch list with DRAM traffic: every kernel of the evaluation
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r02_launches_c3.csv $CMD > gpurun_out/r02_ncu_list.log 2>&1
echo "list rc=$?"
# --set full of the kernel classes (a few launches each, past the first steps)
for spec in "jacobi_cluster:6:1" "jacobi_cluster:60:1" "bqr_panel:10:1" "bq_panel|bq_pick:10:2" "gen_tiles:0:1" \
            "potrf_block:20:1" "trsm_vbatch:20:1" "sumsq:10:1" "copy_kernel:20:1"; do
  IFS=: read -r re skip cnt <<< "$spec"
  tag=$(echo "$re" | cut -d'|' -f1)_$skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$re" -s $skip -c $cnt \
      -o gpurun_out/r02_full_$tag $CMD > gpurun_out/r02_ncu_full_$tag.log 2>&1
  echo "$tag rc=$?"
done
# the GEMM tile configurations by their demangled names: 64 x 64 two-stage (default), thin, small
for spec in "dgemm_tiles_kernel<.int.64, .int.64, .int.32, .int.32, .int.2,:300:2:gemm64" \
            "dgemm_tiles_kernel<.int.32, .int.32,:50:1:gemm_small"; do
  IFS=: read -r re skip cnt tag <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$re" \
      -s $skip -c $cnt -o gpurun_out/r02_full_$tag $CMD > gpurun_out/r02_ncu_full_$tag.log 2>&1
  echo "$tag rc=$?"
done
# dense C3: the trailing-update GEMM (FP64 tensor pipe), the blocked TRSM's diagonal solves, POTRF
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_tiles -s 60 -c 3 \
    -o gpurun_out/r02_full_dense_gemm python tools/trace_cfg.py C3 --no-warm --dense > gpurun_out/r02_ncu_full_dense_gemm.log 2>&1
echo "dense gemm rc=$?"
gzip -f gpurun_out/r02_launches_c3.csv
python tools/ncu_rep_table.py gpurun_out/r02_full_*.ncu-rep > gpurun_out/r02_counters.md 2>&1
cat gpurun_out/r02_counters.md | cut -c1-250
# the merge back is capped at 64 MiB: drop the largest reports beyond 50 MB (their counters are in r02_counters.md)
while [ $(du -sm gpurun_out | cut -f1) -gt 50 ]; do
  big=$(ls -S gpurun_out/*.ncu-rep | head -1); echo "dropping $big"; rm -f "$big"
done
ls -la gpurun_out/

# round-2 profiles: ncu --set full of the dominant kernel (config 4 matvec) and
# the launch list of one bench step (50-iteration BD-GMRES, config 4)
set -x
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_dlp_sym -c 1 \
  -f -o $O/k_dlp_sym_r2 python tools/ncu_step.py matvec 4 > $O/ncu_sym.log 2>&1; echo "ncu sym rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_step_config4_r2.csv python tools/ncu_step.py step 4 > $O/ncu_step.log 2>&1; echo "ncu step rc=$?"
python tools/ncu_summary.py $O/k_dlp_sym_r2.ncu-rep > $O/k_dlp_sym_r2_summary.txt 2>&1
python tools/summarize_launches.py $O/launches_step_config4_r2.csv > $O/launches_step_config4_r2_summary.txt 2>&1
cat $O/k_dlp_sym_r2_summary.txt $O/launches_step_config4_r2_summary.txt

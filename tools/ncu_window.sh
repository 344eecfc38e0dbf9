cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
export DR_LIB_VARIANT=L1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_sl_window.*EpiIncState" -s 6 -c 1 -o gpurun_out/win_L1 $CMD > gpurun_out/win_L1.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/win_L1.ncu-rep --page raw --csv > gpurun_out/win_L1_raw.csv 2>/dev/null
ncu -i gpurun_out/win_L1.ncu-rep --page details --csv > gpurun_out/win_L1_details.csv 2>/dev/null
ncu -i gpurun_out/win_L1.ncu-rep --page source --csv > gpurun_out/win_L1_source.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/win_L1.ncu-rep > gpurun_out/win_L1_summary.txt 2>&1
unset DR_LIB_VARIANT
export DR_WINDOW=0
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_sl_gather.*EpiIncState" -s 6 -c 1 -o gpurun_out/pair_r2 $CMD > gpurun_out/pair_r2.log 2>&1
python tools/ncu_summary.py gpurun_out/pair_r2.ncu-rep > gpurun_out/pair_r2_summary.txt 2>&1
ncu -i gpurun_out/pair_r2.ncu-rep --page raw --csv > gpurun_out/pair_r2_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out

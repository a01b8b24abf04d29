# steady-state ncu launch list + full capture of one cfg2 fine step (tools/ncu_one.py)
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_one.py graphs=0 > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"fft_lanes|leg_synth_v3|leg_anal_v3|k_helm_tiled|k_cn_fused|k_cn_decide|k_cn_finish" -c 14 -o gpurun_out/full python tools/ncu_one.py graphs=0 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?

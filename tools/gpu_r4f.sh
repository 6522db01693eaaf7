# round 2, final ncu artefacts at HEAD (box 28): launch list of the bench command, --set full of one solve application and of the full factorisation on c4
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4f_launches_c4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > gpurun_out/r4f_ncu.log 2>&1; echo "ncu rc $?" >> gpurun_out/r4f_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_line_solve_rt -s 4 -c 1 -o gpurun_out/r4f_rt_c4 python tools/profile_case.py c4 0 > gpurun_out/r4f_ncu_rt.log 2>&1
bash tools/ncu_summary.sh gpurun_out/r4f_rt_c4.ncu-rep > gpurun_out/r4f_rt_c4_summary.txt
timeout 900 ncu --set full --clock-control none -k regex:k_line_factor -c 1 -o gpurun_out/r4f_factor_c4 python tools/profile_case.py c4 0 > gpurun_out/r4f_ncu_factor.log 2>&1
bash tools/ncu_summary.sh gpurun_out/r4f_factor_c4.ncu-rep > gpurun_out/r4f_factor_c4_summary.txt
rm -f gpurun_out/r4f_factor_c4.ncu-rep gpurun_out/r4f_rt_c4.ncu-rep
tail -2 gpurun_out/r4f_ncu.log | cut -c1-300; cat gpurun_out/r4f_rt_c4_summary.txt | head -12; cat gpurun_out/r4f_factor_c4_summary.txt | head -8

# round 2 final captures (box 18): GPU suite, smoke, default bench + reference arm, bench lines of c1/c2/c3/c5,
# ncu launch list of the bench command, ncu --set full of the factor on c4
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -x -q -m gpu --durations=8 ) > gpurun_out/r3s_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r3s_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3s_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r3s_smoke.log
( time timeout 900 python bench.py ) > gpurun_out/r3s_bench_c4.json 2> gpurun_out/r3s_bench_c4.err; echo "bench rc $?" >> gpurun_out/r3s_bench_c4.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/r3s_ref_c4.json 2> gpurun_out/r3s_ref_c4.err; echo "ref rc $?" >> gpurun_out/r3s_ref_c4.err
for c in c3 c5 c2 c1; do
  timeout 900 python bench.py --config $c > gpurun_out/r3s_bench_$c.json 2> gpurun_out/r3s_bench_$c.err; echo "bench $c rc $?" >> gpurun_out/r3s_bench_$c.err
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3s_launches_c4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variants > gpurun_out/r3s_ncu.log 2>&1; echo "ncu rc $?" >> gpurun_out/r3s_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_line_factor -c 1 -o gpurun_out/r3s_factor_c4 python tools/profile_case.py c4 0 > gpurun_out/r3s_ncu_factor.log 2>&1
bash tools/ncu_summary.sh gpurun_out/r3s_factor_c4.ncu-rep > gpurun_out/r3s_factor_c4_summary.txt
rm -f gpurun_out/r3s_factor_c4.ncu-rep
tail -12 gpurun_out/r3s_pytest.log; cat gpurun_out/r3s_smoke.log; for f in gpurun_out/r3s_bench_*.json gpurun_out/r3s_ref_c4.json; do echo $f; cut -c1-160 $f; done; tail -2 gpurun_out/r3s_ncu.log; cat gpurun_out/r3s_factor_c4_summary.txt | head -30

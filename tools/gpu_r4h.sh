# round 2, final validation after the robustness fixes (box 30, final HEAD): GPU suite twice, smoke, default bench, reference arm, c1/c2/c3/c5 lines
for i in 1 2; do ( time timeout 1500 python -m pytest tests -x -q -m gpu ) > gpurun_out/r4h_pytest_$i.log 2>&1; echo "pytest $i rc $?" >> gpurun_out/r4h_pytest_$i.log; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4h_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r4h_smoke.log
( time timeout 900 python bench.py ) > gpurun_out/r4h_bench_c4.json 2> gpurun_out/r4h_bench_c4.err; echo "bench rc $?" >> gpurun_out/r4h_bench_c4.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/r4h_ref_c4.json 2> gpurun_out/r4h_ref_c4.err; echo "ref rc $?" >> gpurun_out/r4h_ref_c4.err
for i in 1 2; do tail -5 gpurun_out/r4h_pytest_$i.log | tr '\n' ' '; echo; done; cat gpurun_out/r4h_smoke.log
for f in gpurun_out/r4h_bench_*.json gpurun_out/r4h_ref_c4.json; do echo $f; cut -c1-130 $f; done

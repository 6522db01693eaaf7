# round 2, session 3: tiled imaging kernels (parity + timing), per-config bench lines c1/c2/c3/c5 at HEAD
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "imaging or data_terms" > gpurun_out/r2af_img.log 2>&1; echo "rc $?" >> gpurun_out/r2af_img.log
for c in c1 c2 c3 c5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2af_bench_$c.json 2> gpurun_out/r2af_bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_smooth|k_terms|k_deriv" -c 20 python tools/profile_case.py c4 0 > gpurun_out/r2af_img_ncu.txt 2>&1
tail -3 gpurun_out/r2af_img.log
for c in c1 c2 c3 c5; do python -c "
import json,sys; d=json.load(open('gpurun_out/r2af_bench_$c.json')); s=d['solver']
print('$c', round(d['value'],4), 'ms', round(d['ms_per_step'],1), 'factor', round(s['ms_factor'],1), 'pcg', round(s['ms_pcg'],1), 'iters', s['pcg_iterations_per_step'], 'frac', round(d['roofline']['frac'],3), d['roofline']['kernel'][:18], 'ffrac', d.get('roofline_factor',{}).get('frac'))"; done
grep -E "k_smooth|k_terms|k_deriv|duration|bytes" gpurun_out/r2af_img_ncu.txt | head -40

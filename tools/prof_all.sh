set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fwd_tile_kernel -s 6 -c 6 -o gpurun_out/r01_fwd_final python tools/prof_forward.py --steps 2 > gpurun_out/ncu_fwd.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:transform_kernel -s 1 -c 1 -o gpurun_out/r01_tr_final python tools/prof_forward.py --steps 2 > gpurun_out/ncu_tr.log 2>&1
python tools/launches_summary.py gpurun_out/r01_bench_launches.csv | head -8
python tools/ncu_json.py gpurun_out/r01_fwd_final.ncu-rep gpurun_out/forward_ncu_summary.json "ncu --set full --clock-control none, tools/prof_forward.py --steps 2 (pop 10k, B=4096), round 1 final kernel" | tail -3

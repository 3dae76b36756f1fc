#!/usr/bin/env bash
# Regenerates the round-2 evidence under profiles/ on a B200 (run via gpurun from the repo root):
# pass ncu capture -> forward_ncu_summary.json (the bench line's roofline.traffic), the bench line,
# the reference arm, the bench launch list and the rollout capture, each profiled command first
# run plainly.  Outputs land in gpurun_out/; copy the summaries into profiles/.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python tools/prof_pass.py --steps 2 > $O/pp.log 2>&1 || exit 3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"transform_kernel|plan_tc|fwd_" -s 9 -c 9 -o $O/r02_pass_final python tools/prof_pass.py --steps 2 > $O/ncu_pass.log 2>&1
python tools/ncu_json.py $O/r02_pass_final.ncu-rep profiles/forward_ncu_summary.json "ncu --set full --clock-control none, tools/prof_pass.py --steps 2 (pop 10k, B=4096): the 2nd step's transform + device-planned tensor-core forward (plan_tc_kernel + 6 fwd_tc_kernel class launches + fwd_tile_kernel), round 2 final kernels" > $O/ncu_json.log 2>&1
cp profiles/forward_ncu_summary.json $O/forward_ncu_summary.json
python tools/ncu_summary.py $O/r02_pass_final.ncu-rep > $O/r02_pass_ncu_summary.txt 2>&1
timeout 600 python bench.py > $O/r02_bench_line.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/r02_reference_arm.json 2> $O/ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-secondary > $O/launch.log 2>&1
timeout 300 python tools/bench_configs.py recurrent --pop 10000 --sweeps 5 --steps 10 --no-cpu > $O/rec_plain.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:rollout -s 1 -c 1 -o $O/r02_rollout_final python tools/bench_configs.py recurrent --pop 10000 --sweeps 5 --steps 10 --no-cpu > $O/rec_ncu.log 2>&1
python tools/ncu_summary.py $O/r02_rollout_final.ncu-rep > $O/r02_rollout_ncu_summary.txt 2>&1
tail -c 400 $O/r02_bench_line.json; echo; tail -c 300 $O/r02_reference_arm.json

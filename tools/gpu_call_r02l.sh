mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
grep -v "^\s*$" gpurun_out/bench.err | tail -5
python -c "import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['c2_step_coarse_to_fine'], d['c2_step_with_mgpcg']['ms_per_step'])"

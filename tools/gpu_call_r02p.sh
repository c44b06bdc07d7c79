mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for uf in s h; do for lv in 1 2; do C3_WS_GB=48 python tools/c3_one.py $lv $uf 100000; done; done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'])
print({k:(round(v['ms'],2), round(v['k4_roofline']['frac'],3)) for k,v in d['c3_cholesky_ir'].items()})
print({k:round(v['ms_alone'],3) for k,v in d['per_level'].items()})"

mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_dd.py -x -q > gpurun_out/pytest_dd.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/pytest_dd.log
timeout 300 python tools/dd_time.py > gpurun_out/dd_time.json 2> gpurun_out/dd_time.err; echo "dd_time rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/dd_time.json'))
for k,v in d.items(): print(k, {kk:(round(vv['us_per_step'],2) if 'us_per_step' in vv else round(vv['ms_coupled_sample'],1)) for kk,vv in v.items() if isinstance(vv,dict)})"
tail -3 gpurun_out/dd_time.err

mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "separable or field" > gpurun_out/pytest_field.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_field.log
for v in sep dense; do
  for a in "C2 0 20000" "C2 1 5000" "C2 2 1200" "C2 3 300" "C3 2 20000" "C5 0 1000000" "C5 2 20000" "C5 4 200" "C5 6 20"; do
    MLMC_FIELD_KERNEL=$v timeout 300 python tools/level_profile.py $a 2>&1 | grep field | sed "s/^/$v /"
  done
done
MLMC_FIELD_KERNEL=sep timeout 300 python tools/level_profile.py C2 3 300 > /dev/null 2>&1 && \
MLMC_FIELD_KERNEL=sep timeout 600 ncu --set full --clock-control none -k regex:field_sep -c 2 --csv --page raw \
  python tools/level_profile.py C2 3 300 > gpurun_out/ncu_sep_raw.csv 2> gpurun_out/ncu_sep.err; echo "ncu rc=$?"
timeout 300 python bench.py --steps 20 --warmup 5 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 step', d['ms_per_step'], d['value'])"

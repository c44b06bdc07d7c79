# A/B: K3 N=64 register cap (co-residency of other levels' CTAs in the C2 step)
mkdir -p gpurun_out
for reg in 0 232 208 192; do
  if [ $reg -gt 0 ]; then export MLMC_K3_MAXREG=$reg; else unset MLMC_K3_MAXREG; fi
  touch paper_2503_05533_b200/csrc/k_minres_tile.cu
  python -c "from paper_2503_05533_b200 import build as b; b.build()" > gpurun_out/build_$reg.log 2>&1 || { tail -5 gpurun_out/build_$reg.log; continue; }
  for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('reg $reg C2', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), [round(v['ms_alone'],3) for v in d['per_level'].values()])"; done
done

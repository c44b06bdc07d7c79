# after the h = 1/8 tile change: full GPU suite (production build), then the per-launch A/B (tuning build)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build_t.log 2>&1 || { tail -30 gpurun_out/build_t.log; exit 1; }
MLMC_TUNING=1 timeout 300 python tools/tune_minres.py 2>&1 | grep '"N": 8'

mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python tools/e1_bias_variance.py gpurun_out/e1.json > gpurun_out/e1.log 2>&1; echo "e1 rc=$?"; tail -6 gpurun_out/e1.log
timeout 900 python tools/paper_experiment.py 1000 gpurun_out/paper_experiment_R1000.json > gpurun_out/paper_exp.log 2>&1; echo "paper rc=$?"; tail -6 gpurun_out/paper_exp.log

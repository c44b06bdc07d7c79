mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
for ws in 4 16 48; do for uf in s h; do for lv in 1 2; do C3_WS_GB=$ws python tools/c3_one.py $lv $uf 100000 | sed "s/^/ws=$ws GB: /"; done; done; done

python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for cs in 2 4; do MLMC_STREAM_CLUSTER=$cs timeout 300 python tools/k3c_cluster.py 6 100 1.9e-7 gpurun_out/l6_cs$cs.npy; done
for n in 100 441; do for cs in 1 2 4 8; do MLMC_STREAM_CLUSTER=$cs timeout 300 python tools/k3c_cluster.py 4 $n 1.4e-5 gpurun_out/l4_cs$cs.npy; done; done
for cs in 1 4; do MLMC_STREAM_CLUSTER=$cs timeout 300 python tools/k3c_cluster.py 5 300 3.4e-6 gpurun_out/l5b_cs$cs.npy; done

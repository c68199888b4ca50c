python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2peak scripts/l2_random_peak.cu && /tmp/l2peak > gpurun_out/l2peak.log 2>&1
DRG_DRAW_ILP=1 timeout 300 python scripts/split_probe.py mesh > gpurun_out/split_probe_ilp1.log 2>&1
DRG_DRAW_ILP=2 timeout 300 python scripts/split_probe.py mesh > gpurun_out/split_probe_ilp2.log 2>&1
timeout 3000 python scripts/quality.py rgg 32 sampled:16:4,sampledf:16:4 gpu 400 > gpurun_out/quality_ab.log 2>&1
cat gpurun_out/l2peak.log; grep level gpurun_out/split_probe_ilp*.log; grep '^{' gpurun_out/quality_ab.log | cut -c1-300

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python scripts/quality.py grid 100 sampled,jacobi gpu 1000 > gpurun_out/quality_grid_final.log 2>&1
timeout 3000 python scripts/quality.py mesh 4 sampled gpu 0 > gpurun_out/quality_mesh_c4.log 2>&1
grep '^{' gpurun_out/quality_grid_final.log | cut -c1-250; grep '^{' gpurun_out/quality_mesh_c4.log | cut -c1-250; tail -n 3 gpurun_out/quality_mesh_c4.log | cut -c1-200

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 bash scripts/profile.sh mesh sampled > gpurun_out/profile_sampled.log 2>&1
cat gpurun_out/profile_sampled.log

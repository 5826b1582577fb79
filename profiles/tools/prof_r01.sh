set -x
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_sweep_flow|k32_|k_solid_stress_csr|k_solid_accel_csr|k_solid_rmap' -c 12 -o gpurun_out/step_full python profiles/tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out

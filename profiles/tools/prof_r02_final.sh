# Final round-2 captures (run under gpurun from the repo root, after the same
# commands exited 0 without ncu).  The .ncu-rep files exceed what gpurun brings
# back, so the raw / source pages are exported here and the reports dropped.
set -x
cd ${GRAFT_REPO_ROOT:-.}
export PATH=/usr/local/cuda/bin:$PATH
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err
# 1. launch list of the bench command (cold-cache, serialised: shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-serial \
    > gpurun_out/ncu_launch.log 2>&1
# 2. full capture of one fp64 and one fp32 inner step, every kernel class
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_sweep_flow|k_solid_(kick|stress|rmap|accel|vmax)|k32_(kick|stress|rmap|accel|vmax)' \
    -c 12 -o gpurun_out/step_full python profiles/tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/step_full.ncu-rep --page raw --csv > gpurun_out/step_full_raw.csv
rm -f gpurun_out/step_full.ncu-rep
# 3. full capture of the outer diffusion step's kernels (membrane leg)
timeout 900 ncu --set full --clock-control none \
    -k regex:'k_por_(prep|flux|mass|post|fluxrate)' -c 7 -o gpurun_out/outer_full \
    python profiles/tools/membrane_only.py > gpurun_out/ncu_outer.log 2>&1
ncu -i gpurun_out/outer_full.ncu-rep --page raw --csv > gpurun_out/outer_full_raw.csv
rm -f gpurun_out/outer_full.ncu-rep
ls -la gpurun_out

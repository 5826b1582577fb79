# Round-2 profile captures (run under gpurun from the repo root).  Each
# command ran without ncu first (bench / tests); nothing printed here is a
# bench number.
set -x
cd ${GRAFT_REPO_ROOT:-.}
export PATH=/usr/local/cuda/bin:$PATH
# 1. launch list of the bench command (cold-cache, serialised: shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu \
    > gpurun_out/ncu_launch.log 2>&1
# 2. full capture of one fp64 and one fp32 inner step, every kernel class
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_sweep_flow|k_solid_(kick|stress|rmap|accel|vmax)|k32_(kick|stress|rmap|accel|vmax)' \
    -c 12 -o gpurun_out/step_full python profiles/tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
# 3. full capture of the outer diffusion step's kernels (membrane leg)
timeout 900 ncu --set full --clock-control none \
    -k regex:'k_por_(prep|flux|mass|post|fluxrate)' -c 7 -o gpurun_out/outer_full \
    python profiles/tools/membrane_only.py > gpurun_out/ncu_outer.log 2>&1
ls -la gpurun_out
# 4. full capture of the reference-order multi-CTA sweep on a 2 M-particle
#    slice (the parity-mode kernel)
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_sweep_serial_grid' -c 1 -o gpurun_out/serial_grid_full \
    python profiles/tools/prof_step.py --sweep serial --precisions 64 --length 4 \
    > gpurun_out/ncu_serial.log 2>&1
ls -la gpurun_out

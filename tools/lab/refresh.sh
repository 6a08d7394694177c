# Round-end style refresh on one box: GPU tests, the bench line, the graph-replay
# launch list and one ncu --set full capture of an iteration's kernels.
#   TAG=r2d bash tools/lab/refresh.sh
TAG=${TAG:-rX}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputest.log 2>&1; tail -3 gpurun_out/${TAG}_gputest.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -c 600 gpurun_out/${TAG}_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu --skip-noshare --no-configs > gpurun_out/${TAG}_ncu_plain.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv 2>&1 | tail -20
IEDD_B200_NO_GRAPH=1 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:"k_fft8|k_apply_dmma|k_scatter|k_iter|k_update" --launch-skip 30 --launch-count 7 -f \
    -o gpurun_out/${TAG}_full python tools/pcg_launches.py > gpurun_out/${TAG}_ncu.log 2>&1; tail -2 gpurun_out/${TAG}_ncu.log

# quick check of a change on the config-5 PCG iteration: pcg parity, two bench runs, kernel launch times
exec > gpurun_out/quick.log 2>&1
python -m pytest tests -m gpu -x -q -k "${TESTK:-pcg or apply}" | tail -2
for rep in 1 2; do
python bench.py --no-cpu --skip-noshare --matvec fft 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/quick_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --skip-noshare > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/quick_launches.csv

# k_apply_dmma2 (balanced n-tile deal) vs k_apply_dmma (IEDD_B200_DMMA_V1=1): parity, bitwise, timing
exec > gpurun_out/dmma2_ab.log 2>&1
python -m pytest tests -m gpu -x -q -k "apply or pcg or Shard or Factor or CBD" | tail -3
python tools/lab/bitwise_ab.py | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v for k,v in d['hashes'].items() if k.startswith('pcg')})"
IEDD_B200_DMMA_V1=1 python tools/lab/bitwise_ab.py | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v for k,v in d['hashes'].items() if k.startswith('pcg')})"
python tools/ab_env.py IEDD_B200_DMMA_V1 3
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/dmma2_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --skip-noshare > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/dmma2_launches.csv | grep dmma

exec > gpurun_out/e2e_ab.log 2>&1
python -m pytest tests -m gpu -x -q -k "pcg or Pcg or Golden or Propert or smoke or numpy or host" 2>&1 | tail -2
echo new; python tools/e2e_breakdown.py | python -c "import json,sys; d=json.load(sys.stdin); print(d['K'], [round(x,4) for x in d['host_ms']], [round(x,4) for x in d['device_ms']], d['host_ms_fit'], d['device_ms_fit'])"
python tools/lab/bitwise_ab.py | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v for k,v in d['hashes'].items() if k.startswith('pcg')})"

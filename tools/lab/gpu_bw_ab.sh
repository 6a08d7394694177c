set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
mkdir -p gpurun_out
python tools/lab/bitwise_ab.py > gpurun_out/bw_new.json 2> gpurun_out/bw_new.err
IEDD_B200_LIB=$PWD/tools/lab/lib_base.so python tools/lab/bitwise_ab.py > gpurun_out/bw_base.json 2> gpurun_out/bw_base.err
python - <<'PY'
import json
a=json.load(open('gpurun_out/bw_new.json'))['hashes']; b=json.load(open('gpurun_out/bw_base.json'))['hashes']
for k in a: print(k, 'SAME' if a[k]==b[k] else 'DIFF', a[k], b[k])
PY
KREGEX=k_fft8 bash tools/lab/ab_lib.sh
cat gpurun_out/ab_lib.log
if [ -n "$NCU_TAG" ]; then
IEDD_B200_NO_GRAPH=1 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_fft8 --launch-skip 6 --launch-count 3 -f -o gpurun_out/$NCU_TAG python tools/pcg_launches.py > gpurun_out/$NCU_TAG.log 2>&1
fi

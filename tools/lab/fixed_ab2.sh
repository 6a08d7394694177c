exec > gpurun_out/fixed_ab2.log 2>&1
python -m pytest tests -m gpu -x -q -k "pcg or Pcg or Determinism or Golden or Propert or Edge" 2>&1 | tail -2
for r in 1 2; do echo new; python tools/lab/fixed_cost.py; echo base; IEDD_B200_LIB=$PWD/tools/lab/lib_base.so python tools/lab/fixed_cost.py; done

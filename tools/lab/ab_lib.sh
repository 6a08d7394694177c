# same-box A/B: tools/lab/lib_base.so (IEDD_B200_LIB) vs the in-tree build, config-5 PCG iteration
exec > gpurun_out/ab_lib.log 2>&1
for rep in 1 2 3; do
for L in base new; do
if [ $L = base ]; then export IEDD_B200_LIB=$PWD/tools/lab/lib_base.so; else unset IEDD_B200_LIB; fi
python bench.py --no-cpu --skip-noshare --matvec fft 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', d['value'], d['ms_per_step'])"
done; done
unset IEDD_B200_LIB
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${KREGEX:-k_scatter} -c 20 --csv python bench.py --no-cpu --skip-noshare --matvec fft --steps 5 2>/dev/null | grep '"' | tail -3 | awk -F'","' '{print "new", $NF}'
IEDD_B200_LIB=$PWD/tools/lab/lib_base.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${KREGEX:-k_scatter} -c 20 --csv python bench.py --no-cpu --skip-noshare --matvec fft --steps 5 2>/dev/null | grep '"' | tail -3 | awk -F'","' '{print "base", $NF}'

# A/B of the scatter batch variants (IEDD_B200_SCAT_G) on the config-5 PCG iteration
exec > gpurun_out/ab.log 2>&1
for rep in 1 2; do for G in ${GS:-2 11 12}; do
IEDD_B200_SCAT_G=$G python bench.py --no-cpu --skip-noshare --matvec fft 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('G=$G', d['value'], d['ms_per_step'], d['e2e']['value'])"
done; done
for G in ${GS:-2 11 12}; do
IEDD_B200_SCAT_G=$G ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_scatter -c 20 --csv python bench.py --no-cpu --skip-noshare --matvec fft --steps 5 2>/dev/null | grep k_scatter | tail -3 | awk -F'","' '{print "G='$G'", $NF}'
done

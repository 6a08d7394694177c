# one ncu --set full capture of the kernels matching KREGEX in a config-5 PCG solve
#   KREGEX=k_apply_dmma2 TAG=dmma2 bash tools/lab/ncu_one.sh
TAG=${TAG:-one}
IEDD_B200_NO_GRAPH=1 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:"${KREGEX:-k_apply_dmma}" --launch-skip ${SKIP:-6} --launch-count ${COUNT:-1} -f \
    -o gpurun_out/${TAG}_full python tools/pcg_launches.py > gpurun_out/${TAG}_ncu.log 2>&1; tail -2 gpurun_out/${TAG}_ncu.log

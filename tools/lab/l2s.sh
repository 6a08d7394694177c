exec > gpurun_out/l2s.log 2>&1
for mb in 17 18 24 28; do echo "setaside $mb"; python tools/ab_env.py IEDD_B200_L2_SETASIDE_MB=$mb 3; done

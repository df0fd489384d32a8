timeout 200 python tools/profile_classes.py 2>&1 | tail -2
bash tools/ab_gemm.sh 2>&1 | sed -n 1,6p

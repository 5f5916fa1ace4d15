for bw in 0 104 108 8; do TDVP_SVD_BW=$bw timeout 300 python microbench.py --svd --svd-n 16,64,128,256,512 2>&1 | grep '"n"'; done

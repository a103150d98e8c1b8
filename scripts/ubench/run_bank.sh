#!/bin/bash
# Register-number (bank class) test of the DFMA operand-read bound; prints DP warp-inst/clk/SM per variant.
set -e
cd "$(dirname "$0")"
W=/tmp/ubench_bank; rm -rf $W; mkdir -p $W
nvcc -gencode arch=compute_100a,code=sm_100a -cubin -o $W/kb.cubin ubench_bank.cu
python ../lab/bank_variants.py $W/kb.cubin $W/var > $W/variants.txt
g++ -O2 -o $W/bank_host bank_host.cpp -I/usr/local/cuda/include -L/usr/local/cuda/lib64/stubs -lcuda
cd $W/var && $W/bank_host orig.cubin $(ls *.cubin | grep -v orig) 

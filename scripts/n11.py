"""Build and run the N11 microbenchmarks (scripts/n11_microbench.cu) on cuda:0; prints JSON lines."""
import os
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
exe = os.path.join("/tmp", "n11_microbench")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                       os.path.join(here, "n11_microbench.cu"), "-o", exe])
sys.exit(subprocess.call([exe]))

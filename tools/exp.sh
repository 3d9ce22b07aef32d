mkdir -p gpurun_out
./tools/microbench > gpurun_out/microbench.log 2>&1
CONCORD_PHASE_PROFILE=1 timeout 300 python tools/profile_fit.py --p 5000 --n 2000 --fits 1 > gpurun_out/phase5000.log 2>&1
CONCORD_PHASE_PROFILE=1 timeout 300 python tools/profile_fit.py --p 1000 --n 500 --fits 1 > gpurun_out/phase1000.log 2>&1
CONCORD_PHASE_PROFILE=1 timeout 300 python tools/profile_fit.py --p 5000 --n 2000 --fits 1 --n-blocks 74 > gpurun_out/phase5000_74.log 2>&1
CONCORD_PHASE_PROFILE=1 timeout 300 python tools/profile_fit.py --p 5000 --n 2000 --fits 1 --lam 0.0 --max-iter 3 > gpurun_out/phase5000_dense.log 2>&1

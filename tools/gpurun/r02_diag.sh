cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for b in 128; do timeout 300 python tools/diag_parity.py cifar_b512 $b 1.48; done > gpurun_out/diag.log 2>&1
cat gpurun_out/diag.log

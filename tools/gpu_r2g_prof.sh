# session-3 profiles at HEAD: launch list + DRAM bytes (gpu_prof2.sh), then a
# source-level capture of the chain and preprocess kernels
set -x
TAG=${TAG:-r2g} bash tools/gpu_prof2.sh
TAG=r2g FULLK="chain_kernel|preprocess_kernel|surfel_prepass" FULLC=3 bash tools/gpu_src_prof.sh
ls -la gpurun_out

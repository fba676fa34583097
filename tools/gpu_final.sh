#!/bin/bash
# final measurement set of the round
bash tools/round_profile.sh r02_final
bash tools/shared_gpu_check.sh r02_final/nproc
bash tools/bounds_run.sh r02_final/bounds
ls gpurun_out/r02_final

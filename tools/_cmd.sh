#!/bin/bash
# scratch driver for one gpurun call
mkdir -p gpurun_out
bash tools/gpu_check.sh tests
bash tools/gpu_check.sh bench

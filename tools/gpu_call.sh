#!/bin/bash
# Scratch runner for one gpurun call: `gpurun -- bash tools/gpu_call.sh '<commands>'`.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
eval "$1"

#!/bin/bash
# Dense-contraction timing + ncu (refresh / oracle / metrics kernels) and
ls -la gpurun_out

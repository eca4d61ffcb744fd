#!/bin/bash
mkdir -p gpurun_out
bash scripts/sanitize.sh

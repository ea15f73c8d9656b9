#!/bin/bash
cd "$(dirname "$0")/.."
bash tools/r2_ncu_kernel.sh tail42p r2_tailp_ncu
bash tools/r2_ncu_kernel.sh fourier128_tc2 r2_k1_ncu

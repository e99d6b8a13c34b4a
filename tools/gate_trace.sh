# Debug build with the gate's %globaltimer phase stamps (MOE_GATE_TRACE) into
# paper_2201_05596_b200/libmoe_b200_trace.so, then the per-phase times of one
# gate launch (CTA 0) at the given token counts: bash tools/gate_trace.sh [--build]
set -e
cd "$(dirname "$0")/.."
if [ "$1" = "--build" ]; then
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -shared --expt-relaxed-constexpr --threads 0 -DMOE_GATE_TRACE -I include \
    -o paper_2201_05596_b200/libmoe_b200_trace.so paper_2201_05596_b200/csrc/*.cu
  exit 0
fi
MOE_B200_LIB=$PWD/paper_2201_05596_b200/libmoe_b200_trace.so python tools/gate_trace.py

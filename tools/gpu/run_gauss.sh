# Gaussian-selector parity tests + the C3 (16 x 128K) in-graph timeline with k_gauss_select phases
make -j4 all > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q -k "gauss or Gauss" 2>&1 | tail -5
bash tools/gpu/run_trace.sh 8 131000 gauss 1 16

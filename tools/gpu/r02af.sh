set -x
for k in bq bk fwd; do
  timeout 300 python tools/trace_kernel.py --kernel $k --cta-table > gpurun_out/trace_$k.txt 2>&1
done

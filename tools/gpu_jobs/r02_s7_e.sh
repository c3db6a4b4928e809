mkdir -p gpurun_out
cp paper_2601_11437_b200/libmaternfisher.so /tmp/lib_default.so
for v in default noinl2 default noinl2; do
  if [ $v = default ]; then cp /tmp/lib_default.so paper_2601_11437_b200/libmaternfisher.so; else cp gpurun_variants/lib_$v.so paper_2601_11437_b200/libmaternfisher.so; fi
  echo "== $v"
  timeout 600 python tools/gen_config4_probe.py config4 2>&1 | grep GENPROBE | python -c "
import json,sys; d=json.loads(sys.stdin.read()[9:]); print({k:round(v,1) for k,v in d.items() if k not in ('bits','workload')})"
  python tools/gen_bench.py 2>&1 | grep "gen GB" | tail -1
done
cp /tmp/lib_default.so paper_2601_11437_b200/libmaternfisher.so

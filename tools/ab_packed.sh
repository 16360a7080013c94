# A/B of the packed-FP32 variants (kk_common.cuh KK_PACKED_*): bench stage
# times per variant build, two interleaved repetitions.
#   bash tools/ab_packed.sh base k2add k2mul ...   (base = the default build)
V=paper_2108_07001_b200/_lib/variants
for r in 1 2; do for v in "$@"; do
  lib=$V/$v/libkkb200_$v.so; [ "$v" = base ] && lib=paper_2108_07001_b200/_lib/libkkb200.so
  echo "== $v rep $r"
  KKB200_LIB=$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-checks --no-64qam --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['ms_per_step'],2), {k: round(v,3) for k,v in d['stage_ms'].items()}, 'e2e', round(d['e2e']['value'],3))"
done; done

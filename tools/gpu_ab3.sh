for rep in 1 2; do
for cfg in "base 1" "default 0" "default 1"; do
  set -- $cfg
  if [ $1 = default ]; then unset PIC_LIB_PATH; else export PIC_LIB_PATH=$PWD/paper_2102_13133_b200/libpic_b200_$1.so; fi
  PIC_BATCH_SPECIES=$2 timeout 900 python bench.py --config thermal --steps 20 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.load(sys.stdin); print('$1 batch=$2', '%.4g' % d['value'], '%.4f' % d['ms_per_step'], 'kr %.4g' % d['config']['push_kernel_rate'], 'frac(kr) %.4f' % (d['config']['push_kernel_rate']*64/6456.8e9), d['clocks']['sm_mhz'])"
done; done

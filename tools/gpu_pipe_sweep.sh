for E in "PIC_PIPE_PUSH=0" "PIC_PIPE_PREFETCH=0" "PIC_PIPE_PREFETCH=1" "PIC_PIPE_PREFETCH=2" "PIC_PIPE_PREFETCH=4"; do
  env $E timeout 900 python bench.py --config thermal --steps 20 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.load(sys.stdin); print('$E', '%.4g' % d['value'], '%.4f' % d['ms_per_step'], 'kr %.4g' % d['config']['push_kernel_rate'], 'frac', round(d['roofline']['frac'],4))"
done

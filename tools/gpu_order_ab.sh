#!/bin/bash
# A/B of the continuous voxel order (PIC_VOXEL_ORDER=1, default) against the
# in-place push + deferred sort (0) on the bench decks; one JSON summary per run.
set -u
out=${1:-gpurun_out/order_ab}
mkdir -p "$(dirname $out)"
for cfg in ${CONFIGS:-two_stream thermal weak}; do
  for vo in 1 0; do
    # thermal (0.35 ms steps): a warm-up of three sort cycles so the step's
    # CUDA graphs (one per host state of the voxel-order cycle) are captured
    steps=20; warm=5; [ $cfg = thermal ] && steps=100 && warm=60
    PIC_VOXEL_ORDER=$vo python bench.py --config $cfg --steps $steps --warmup $warm --no-cpu-baseline --no-e2e \
      > ${out}_${cfg}_vo${vo}.json 2>> ${out}.log
    python - "$cfg" "$vo" "${out}_${cfg}_vo${vo}.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[3])); c = d["config"]
print(f"{sys.argv[1]:>10} vo={sys.argv[2]} value {d['value']:.3e} ms/step {d['ms_per_step']:.3f} push {c['push_kernel_rate']:.3e} "
      f"frac {d['roofline']['frac']:.3f} clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']} "
      f"phases {{{', '.join(f'{k}: {v:.3f}' for k, v in c['phase_ms_per_step'].items())}}}")
PY
  done
done

#!/bin/bash
# C2 N=1 step time with one piece of work removed at a time (PP200_ABLATE /
# PP200_ABLATE_BIAS_GRAD): how much of the step each piece accounts for.
run() {
  tag=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/abl_$tag.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/abl_$tag.json').read().splitlines()[-1]);print('$tag', d['ms_per_step'], d['clocks']['sm_mhz'])"
}
run base A=1
run attn_fwd PP200_ABLATE=attn_fwd
run attn_bwd PP200_ABLATE=attn_bwd
run wgrad PP200_ABLATE=wgrad
run lnp PP200_ABLATE=lnp
run bias PP200_ABLATE_BIAS_GRAD=1
run wgrad_bias_lnp PP200_ABLATE=wgrad,lnp PP200_ABLATE_BIAS_GRAD=1
run base2 A=1

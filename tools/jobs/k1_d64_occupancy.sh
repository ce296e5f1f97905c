# K1 at d = 64 (BASELINE config 3): CTAs per SM 3 / 4 / 5 (TKV_K1_MINB64), bench line each
set -x
TAG=${TAG:-r02}
for m in 3 4 5; do
  TKV_K1_MINB64=$m timeout 900 python bench.py --no-cpu --config 3 > gpurun_out/${TAG}_c3_minb$m.json 2> gpurun_out/${TAG}_c3_minb$m.err
  echo "minb $m rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_c3_minb$m.json')); print('minb $m', round(d['value']), round(d['tpot_ms'],4), d['breakdown_ms_per_step']['attend_ms'], round(d['roofline']['frac'],3), d['parity'] if 'parity' in d else '')"
done

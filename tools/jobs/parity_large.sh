# large-sample parity at BASELINE configs 2, 3, 4
set -x
TAG=${TAG:-r02}
for spec in "2::128" "3::64" "4::64"; do
  c=${spec%%::*}; u=${spec#*::}
  timeout 2400 python tools/parity_units.py --config $c --units $u > gpurun_out/${TAG}_parity_c${c}.json 2> gpurun_out/${TAG}_parity_c${c}.err; echo "c$c rc=$?"
  tail -c 400 gpurun_out/${TAG}_parity_c${c}.json; tail -3 gpurun_out/${TAG}_parity_c${c}.err
done

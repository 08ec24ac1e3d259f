# per-sweep time under environment switches: gpu_env_var.sh "NAME:VAR=V,VAR2=V" ...
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  for c in config1 config2; do
    env $(echo $envs | tr ',' ' ') timeout 300 python scripts/sweep_rate.py $c > gpurun_out/ev_${name}_$c.json 2> gpurun_out/ev_${name}_$c.err
  done
done

for d in 192 96 48 24 104 52 26 256 128 64 32; do
  SLAB_PLANE_DEBUG=1 python tools/kernel_microbench.py --dims $d $d $d --reps 30 2>&1 | grep -E "gs_planes kind [012]|variant" | sort | uniq | sed -E "s/.*variant\": \"([^\"]*)\".*gs_sym_ms\": ([0-9.]*).*/  sweep_ms \2/" | cut -c1-120
done

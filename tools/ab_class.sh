# A/B of libvb variants (tools/build_variant.py) on the class-variant assembly
mkdir -p gpurun_out
for v in "$@"; do echo $v; VB_LIBVB=tools/variants/$v.so python tools/time_class.py --meshes kuhn128 --reps 100; done > gpurun_out/ab_class.log 2>&1

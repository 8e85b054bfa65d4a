# DESIGN.md R20 study: PAPER.md Table 2 self-convergence (direct sums, 1/h = 16 ... 128) for the cross-point
# interpolation stencil of the default library (degree 4, radius 3.5 h) and build/interp/*.so variants
mkdir -p gpurun_out
timeout 900 python tools/twodrop_table2.py gpurun_out/td_interp_d4r35.json 16 32 64 128 > gpurun_out/td_interp_d4r35.log 2>&1; echo "default rc=$?"
for lib in build/interp/*.so; do
  n=$(basename $lib .so); n=${n#libstokes_er_}
  STOKES_ER_LIB=$PWD/$lib timeout 900 python tools/twodrop_table2.py gpurun_out/td_interp_$n.json 16 32 64 128 > gpurun_out/td_interp_$n.log 2>&1; echo "$n rc=$?"
done

# Round-2 final evidence on one B200, two gpurun calls:
#   bash tools/r2_final_a.sh TAG   full -m gpu suite + smoke, default bench line (cfg4, 20 steps), reference arm
#   bash tools/r2_final_b.sh TAG   cfg2 / cfg3 / cfg5 lines, bounds-assert builds as memory checker (build them first:
#                                  tools/build_variant.sh assert -DHEB_DEVICE_ASSERT=1, intonly_assert, intonly -- see
#                                  tools/assert_check.sh), cfg4 launch list with DRAM counters, ncu --set full of both
#                                  fused-ModUp engine launches and of the conv
T=${1:-r2z}
bash tools/r2_final_a.sh $T
bash tools/r2_final_b.sh $T

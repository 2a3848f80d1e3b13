#!/bin/bash
L=paper_2508_19140_b200/libinpc_raster.so
cp $L /tmp/new.so
for v in A M; do
  case $v in A) cp paper_2508_19140_b200/libinpc_raster_head.so $L;; M) cp paper_2508_19140_b200/libinpc_raster_mid.so $L;; esac
  bash tools/ncu_quick.sh ${K:-k_blend_fwd} $v | grep -v "occupancy_limit"
done
cp /tmp/new.so $L

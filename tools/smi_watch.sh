#!/bin/bash
# sample SM clock / throttle reasons / power every 200 ms into $1 until killed
while true; do nvidia-smi --query-gpu=timestamp,clocks.sm,clocks_throttle_reasons.active,power.draw,temperature.gpu --format=csv,noheader >> "$1"; sleep 0.2; done

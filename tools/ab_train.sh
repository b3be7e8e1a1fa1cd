#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/probe_train.py > gpurun_out/train_probe.log 2>&1

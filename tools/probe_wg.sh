#!/bin/bash
P="python tools/kernel_probe.py"
$P conv_wgrad 1 96 96 96 128 128
$P conv_wgrad 1 96 96 96 64 128
$P conv_wgrad 1 48 48 48 256 256
$P conv_wgrad 1 192 192 192 64 64

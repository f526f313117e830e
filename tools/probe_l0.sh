#!/bin/bash
P="python tools/kernel_probe.py"
$P conv_fwd 1 192 192 192 64 64
$P conv_dgrad 1 192 192 192 64 64
$P conv_fwd 1 192 192 192 128 64
$P conv_dgrad 1 192 192 192 128 64

#!/bin/bash
# fixed + marginal cost of every kernel family at the BASELINE widths (tools/probes/fixed_cost.py, product library)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L="base:@paper_2406_16282_b200/liblmbp.so"
P="timeout 600 python tools/probes/fixed_cost.py --variants $L --iters 40"
{
$P --norm ln --dtype bf16 --cols 768 --rows 3152,6304,12608,25216,50432 --kernels nfwd,nbwd | sed 's/^/{"survey": "c2_norm", /; s/, {/, /' 
$P --act gelu --dtype bf16 --cols 3072 --rows 3152,6304,12608,25216,50432 --kernels fwd,bwd | sed 's/^/{"survey": "c2_act", /; s/, {/, /'
$P --norm rms --dtype bf16 --cols 4096 --rows 2048,4096,8192,16384 --kernels nfwd,nbwd | sed 's/^/{"survey": "c4_norm", /; s/, {/, /'
$P --dtype bf16 --cols 11008 --rows 1024,2048,4096,8192 --kernels swf,swb | sed 's/^/{"survey": "c4_swiglu", /; s/, {/, /'
$P --act gelu --dtype f32 --cols 3072 --rows 4096,8192,16384,32768 --kernels fwd,bwd | sed 's/^/{"survey": "c3_act", /; s/, {/, /'
$P --norm ln --dtype f32 --cols 768 --rows 4096,8192,16384,32768 --kernels nfwd,nbwd | sed 's/^/{"survey": "c3_norm", /; s/, {/, /'
} > gpurun_out/fixed_cost_survey.jsonl 2> gpurun_out/fixed_cost_survey.err
grep '"fit"' gpurun_out/fixed_cost_survey.jsonl; tail -3 gpurun_out/fixed_cost_survey.err

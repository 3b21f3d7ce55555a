// af_llama.cuh -- bs=1 decode kernels of the Llama-shaped block (filled in below).
#pragma once
#include "af_common.cuh"

// glm_b200.cu — single translation unit for libglm_b200.so (sm_100a).
// The pieces share device symbols (the xorshift jump table) without -rdc.
#include "prng.cu"
#include "scd.cu"
#include "objective.cu"
#include "data.cu"
#include "api.cu"
#include "stream.cu"
#include "peer.cu"
#include "ingest.cu"
#include "chunkfile.cu"

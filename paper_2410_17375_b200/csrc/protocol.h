// protocol.h -- launch interface of the protocol kernels.
#pragma once
#include <cuda_runtime.h>

#include "internal.h"

namespace amusd {

enum {
  kDraftBegin = 0, kDraftEnd, kVerifyBegin, kVerifyEnd, kArBegin, kArEnd,
  kSyncRoundBegin, kSyncDraftBegin, kSyncDraftEnd, kSyncVerifyBegin, kSyncVerifyEnd
};

cudaError_t proto_launch(int which, const ProtoArgs& a, cudaStream_t st, int arg = 0);
cudaError_t launch_session_reset(const ProtoArgs& a, const int* prompt_dev, unsigned long long coin_seed,
                                 cudaStream_t st);
cudaError_t launch_hash_forward(StepCtl* c, unsigned long long* h, int vocab, int eos, int excl, int agree, int always,
                                unsigned long long thr, const int* script, int script_len, int eos_pos,
                                cudaStream_t st);
cudaError_t launch_hash_seed(unsigned long long* h, unsigned long long seed, cudaStream_t st);

}  // namespace amusd

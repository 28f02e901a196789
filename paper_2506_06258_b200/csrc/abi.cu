// C-ABI plumbing: error reporting and version (include/market_eq_b200.h).
#include <stdio.h>

#include "mq_common.cuh"

namespace mq {

static thread_local char g_err[512] = "";

int set_error(cudaError_t e, const char *where) {
    snprintf(g_err, sizeof(g_err), "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
    return -(int)e;
}

int check_launch(const char *where) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(e, where);
    return 0;
}

}  // namespace mq

extern "C" {

const char *mq_last_error(void) { return mq::g_err; }

int mq_abi_version(void) { return MQ_ABI_VERSION; }

}  // extern "C"

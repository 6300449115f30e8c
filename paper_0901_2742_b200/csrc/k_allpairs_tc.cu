// k_allpairs_tc.cu — K5: all-pairs on tcgen05 tensor cores (placeholder until the kernel lands).
#include "sad_internal.cuh"

namespace sad {
bool tc_supported(std::string &why) {
    why = "tcgen05 all-pairs kernel not built yet";
    return false;
}
int launch_allpairs_tc(const AllPairsArgs &, cudaStream_t, std::string &err) {
    err = "not built";
    return -1;
}
}  // namespace sad

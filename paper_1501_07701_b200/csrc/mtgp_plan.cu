// mtgp_plan.cu -- v2 planner (stub until the warp-team kernel lands).
#include "mtgp_plan.h"

namespace mtgpb {

struct PlannerImpl {
    std::vector<mtgp_params> sets;
    int num_sms = 148;
};

Planner::Planner(const std::vector<mtgp_params>& sets, int num_sms) : impl_(new PlannerImpl) {
    impl_->sets = sets;
    impl_->num_sms = num_sms;
}
Planner::~Planner() = default;

bool Planner::v2_supported() const { return false; }

cudaError_t Planner::run(PlanRun&, std::string& err) {
    err = "v2 kernel not available";
    return cudaSuccess;
}

cudaError_t Planner::skip(const DevParams*, uint32_t*, uint64_t, cudaStream_t, std::string& err) {
    err = "skip not available";
    return cudaSuccess;
}

}  // namespace mtgpb

// k_fused_mixed.cu -- mixed-precision fused training kernel (placeholder until
// the tensor-core path lands; build_cfg rejects precision == 1 meanwhile).
#include "romap_internal.cuh"

bool fused_mixed_available() { return false; }

void launch_fused_mixed(const LaunchCtx&, const CfgDev&, const ObjDev*, const RayRec*, int, double*, int*, float*) {}

// TEMPORARY: symbols not implemented yet (removed as the real ones land).
#include "common.cuh"
using namespace spb;
extern "C" size_t spb_lobpcg_workspace(int, int32_t, int32_t) { return 0; }
extern "C" int spb_lobpcg_solve(const spb_operator*, int, const double*, const spb_solver_config*,
                                spb_iter_cb, spb_refill_cb, spb_precond_cb, void*, void*, size_t,
                                double*, double*, double*, uint8_t*, int64_t*, void*) {
  set_error("not implemented");
  return SPB_ERR_CUDA;
}
extern "C" int spb_lobpcg_result_block(int, int32_t, int32_t, void*, void**, int64_t*) {
  return SPB_ERR_CUDA;
}
extern "C" size_t spb_sygv_workspace(int32_t) { return 0; }
extern "C" int spb_sygv(const double*, const double*, int32_t, int32_t, double*, double*, void*,
                        size_t, void*) {
  return SPB_ERR_CUDA;
}
extern "C" size_t spb_assign_workspace(int32_t, int32_t) { return 0; }
extern "C" int spb_assign_qrcp(int, const void*, int64_t, int32_t, int32_t, void*, size_t,
                               int32_t*, int32_t*, double*, void*) {
  return SPB_ERR_CUDA;
}

// The 16-warp build of query.cu (one 512-thread CTA per SM) for fronts of batches with at most one
// query per SM; see launch_query at the end of query.cu.
#define SOFA_QTHREADS 512
#define SOFA_QNS q512
#include "query.cu"

// bulk.cu — placeholder translation unit for the TMA bulk-copy commit pipeline.
#include "kernels.h"

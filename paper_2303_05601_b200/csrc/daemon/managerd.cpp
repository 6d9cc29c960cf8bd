// gfx_managerd: the per-B200 GPU Manager daemon (N1). Started by the cluster
// coordinator (gfx_cluster_create with spawn = 1) as
//     gfx_managerd <shm name> <gpu index>
// or run in-process by a rank via gfx_managerd_serve. See csrc/capi/cluster.cu.
#include <cstdio>
#include <cstdlib>

#include "gpufaas_b200.h"

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: %s <shm name> <gpu index>\n", argv[0]);
        return 2;
    }
    return gfx_managerd_serve(argv[1], std::atoi(argv[2]));
}
